"""Drop-in for the exact branch of xcmix.evaluation.predict_topk
(evaluation.py:121-142): the query is embedded by the reference's own encoder
(outside the B200 path) and ranked against every classifier row by the fused
MIPS kernel (anns.query_topk_batch). The graph-index branch is handed back to
the reference implementation recorded by install().
"""

from __future__ import annotations

import numpy as np

from . import anns
from .errors import ConfigError

_reference_predict = None  # set by install()


def predict_topk(encoder, bank_or_index, query_row, k: int, mode: str = "exact", query_beam: int = 128):
    if mode == "exact":
        from xcmix.encoder import embed  # the caller's encoder (not on the B200 path)

        bank = bank_or_index
        if k > bank.n_labels:
            raise ConfigError("k exceeds the label count")
        emb = embed(encoder, query_row)
        index = getattr(bank, "_astra_index", None)
        if index is None or index.vectors is not bank.weights:
            # a read-only view of the live weights (no finiteness check: the
            # reference scores whatever the bank holds)
            index = anns.AnnsIndex(kind="exact", vectors=bank.weights, snapshot_epoch=0)
            try:
                bank._astra_index = index
            except AttributeError:
                pass
        ids, scores = anns.query_topk_batch(index, np.asarray(emb, dtype=np.float64)[None, :], k)
        return anns.ScoredLabels(ids[0], scores[0])
    if mode == "anns":
        return anns.query_topk(bank_or_index, np.asarray(embed_query(encoder, query_row)), k, query_beam)
    raise ConfigError(f"unknown prediction mode {mode!r}")


def embed_query(encoder, query_row):
    from xcmix.encoder import embed

    return embed(encoder, query_row)
