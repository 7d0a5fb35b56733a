"""Drop-in for the exact (MIPS) branches of xcmix.evaluation:

  predict_topk(encoder, bank, query_row, k, mode="exact")   evaluation.py:121-142
  evaluate(dataset, encoder, bank, ks, mode="exact", ...)    evaluation.py:145-206

The queries are embedded by the reference's own encoder (outside the B200
path) and ranked against every classifier row by the fused exact MIPS kernel
(astra_refresh_topk, fp32-exact mode: descending score, ties to the lower id
= the reference's stable argsort of -scores), batched over all queries,
against the bank's live device weights (bank.device_weights: the drop-in's
device copy while it trains the bank, else an upload per call — no cached
copy that in-place training updates could leave stale). The metric
aggregation is the reference's own functions. Graph-index modes are handed
back to the reference implementations recorded by install().
"""

from __future__ import annotations

import numpy as np

from . import _backend, anns
from .bank import device_weights
from .errors import ConfigError

_reference_predict = None  # set by install()
_reference_evaluate = None  # set by install()
QUERY_CHUNK = 1 << 16


def exact_topk(emb, bank, k: int) -> tuple[np.ndarray, np.ndarray]:
    """(ids int64 [n, k], scores float64 [n, k]) of every embedding row
    against all classifier rows: one batched fp32-exact MIPS launch per chunk."""
    import torch

    ops = _backend.get()
    W = device_weights(bank)
    E = np.ascontiguousarray(np.atleast_2d(emb), dtype=np.float32)
    n = E.shape[0]
    ids = np.empty((n, k), dtype=np.int64)
    scores = np.empty((n, k), dtype=np.float64)
    for lo in range(0, n, QUERY_CHUNK):
        hi = min(n, lo + QUERY_CHUNK)
        ip = torch.zeros(hi - lo + 1, dtype=torch.int64, device=W.device)
        pid = torch.zeros(0, dtype=torch.int32, device=W.device)
        _, top, sc = ops.refresh_topk(torch.from_numpy(E[lo:hi]).to(W.device), ip, pid, k, "fp32", labels_f32=W)
        ids[lo:hi] = top.cpu().numpy()
        scores[lo:hi] = sc.cpu().numpy()
    return ids, scores


def predict_topk(encoder, bank_or_index, query_row, k: int, mode: str = "exact", query_beam: int = 128):
    if mode == "exact":
        from xcmix.encoder import embed  # the caller's encoder (not on the B200 path)

        bank = bank_or_index
        if k > bank.n_labels:
            raise ConfigError("k exceeds the label count")
        emb = embed(encoder, query_row)
        ids, scores = exact_topk(np.asarray(emb, dtype=np.float32)[None, :], bank, k)
        return anns.ScoredLabels(ids[0], scores[0])
    if mode == "anns":
        return anns.query_topk(bank_or_index, np.asarray(embed_query(encoder, query_row)), k, query_beam)
    raise ConfigError(f"unknown prediction mode {mode!r}")


def embed_query(encoder, query_row):
    from xcmix.encoder import embed

    return embed(encoder, query_row)


def evaluate(dataset, encoder, bank, ks=(1, 3, 5), mode: str = "exact", propensity=None, anns_params=None):
    """Aggregate the metrics over the split's rows with nonempty positives
    (evaluation.py:145-206); the exact ranking (evaluation.py:163-166: the
    full emb @ W^T score matrix + a stable argsort) is one batched top-kmax
    MIPS pass on the GPU."""
    import xcmix.evaluation as xe
    from xcmix.encoder import embed_batch

    if mode != "exact":
        if _reference_evaluate is None:
            raise ConfigError(f"evaluation mode {mode!r} is not served by the B200 path")
        return _reference_evaluate(dataset, encoder, bank, ks=ks, mode=mode, propensity=propensity,
                                   anns_params=anns_params)
    ks = tuple(sorted(set(int(k) for k in ks)))
    if ks[-1] > dataset.n_labels:
        raise ConfigError("k exceeds the label count")
    if ks[-1] > 2048:
        raise ConfigError("exact GPU evaluation supports k <= 2048")
    if propensity is None:
        stats = dataset.stats()
        propensity = xe.fit_propensity(stats.label_frequency, max(dataset.n_points, 2))
    emb = embed_batch(encoder, dataset.features)
    ranked_all, _ = exact_topk(emb, bank, ks[-1])
    report = xe.MetricsReport(p_at={k: 0.0 for k in ks}, ndcg_at={k: 0.0 for k in ks}, psp_at={k: 0.0 for k in ks},
                              psn_at={k: 0.0 for k in ks})
    for i in range(dataset.n_points):
        pos = dataset.positives[i]
        if len(pos) == 0:
            report.n_excluded += 1
            continue
        report.n_evaluated += 1
        ranked = ranked_all[i]
        for k in ks:
            report.p_at[k] += xe.precision_at_k(ranked, pos, k)
            report.ndcg_at[k] += xe.ndcg_at_k(ranked, pos, k)
            report.psp_at[k] += xe.psp_at_k(ranked, pos, propensity, k)
            report.psn_at[k] += xe.psn_at_k(ranked, pos, propensity, k)
    if report.n_evaluated:
        for table in (report.p_at, report.ndcg_at, report.psp_at, report.psn_at):
            for k in ks:
                table[k] /= report.n_evaluated
    return report
