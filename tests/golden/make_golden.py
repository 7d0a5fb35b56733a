"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Runs only in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It drives the reference's own functions (xcmix.trainer._batch_forward_backward,
xcmix.trainer._assemble_batch_slates, xcmix.anns.retrieve_hard_negatives,
xcmix.classifiers.apply_classifier_updates_arrays) on seeded synthetic inputs
and records their inputs and outputs. Recording is done by wrapping the
module globals the trainer resolves at call time (trainer.py:364, :385,
:394), so the reference code itself runs unmodified.

The fixtures pin oracle/xcmix_port.py (tests/test_oracle_golden.py); the
oracle then checks the CUDA path at any size. Nothing here runs on the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import xcmix.anns as anns
import xcmix.classifiers as classifiers
import xcmix.trainer as trainer
from xcmix.dataset import SparseDataset

HERE = os.path.dirname(os.path.abspath(__file__))


def _dataset(n, D, L, seed, min_pos=1, max_pos=6, first_row_pos=1):
    rng = np.random.default_rng(seed)
    feats = sp.random(n, D, density=0.2, format="csr", dtype=np.float32, random_state=np.random.RandomState(seed))
    positives = []
    for i in range(n):
        k = first_row_pos if i == 0 else int(rng.integers(min_pos, max_pos + 1))
        positives.append(np.sort(rng.choice(L, size=k, replace=False)).astype(np.int32))
    return SparseDataset(n, D, L, feats, positives)


def _csr(positives):
    indptr = np.zeros(len(positives) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(p) for p in positives])
    ids = np.concatenate([np.asarray(p, dtype=np.int32) for p in positives]) if len(positives) else np.zeros(0, np.int32)
    return indptr, ids


def make_step_fixture(name, *, L, d, n, B, k_p, k_h, k_r, dropout, n_steps, seed, wd=1e-3):
    ds = _dataset(n, d, L, seed)
    cfg = trainer.TrainConfig(
        epochs=4, batch_size=B, lr_encoder=0.01, lr_classifier=0.5, warmup_steps=1,
        dropout=dropout, weight_decay_classifier=wd, k_r=k_r, k_h=k_h, k_p=k_p,
        tau_s=2, tau_r=2, strategy="Mixture", embed_dim=d, seed=seed,
    )
    state = trainer.TrainerState(ds, cfg)
    emb_all = trainer.embed_batch(state.encoder, ds.features)
    cache = anns.retrieve_hard_negatives(anns.build_exact(state.bank.weights), emb_all, ds.positives, k_h)
    state.caches.negative_cache = cache

    rec = {}
    orig_asm = trainer._assemble_batch_slates
    orig_enc = trainer.encoder_backward_batch
    orig_upd = trainer.apply_classifier_updates_arrays

    def asm(state_, batch_rows, epoch, rng, hard_batch):
        out = orig_asm(state_, batch_rows, epoch, rng, hard_batch)
        rec["slates"] = out
        rec["hard_batch"] = None if hard_batch is None else hard_batch.copy()
        return out

    def enc(params, rows, G):
        rec["grad_emb"] = np.array(G, copy=True)
        return orig_enc(params, rows, G)

    def upd(bank, ids, grads, lr, wd_):
        rec["uids"] = np.array(ids, copy=True)
        rec["grads"] = np.array(grads, copy=True)
        rec["lr"] = lr
        return orig_upd(bank, ids, grads, lr, wd_)

    trainer._assemble_batch_slates, trainer.encoder_backward_batch, trainer.apply_classifier_updates_arrays = asm, enc, upd
    out = {"L": L, "d": d, "k_p": k_p, "k_h": k_h, "k_r": k_r, "wd": wd, "dropout": dropout, "n_steps": n_steps}
    try:
        epoch = 3  # hard-negative regime (epoch >= tau_s)
        rng = np.random.default_rng((seed, 7919, epoch))
        rows = state.active_rows[rng.permutation(len(state.active_rows))]
        for t in range(n_steps):
            batch = rows[t * B : (t + 1) * B]
            feats = ds.features[batch]
            emb = trainer.embed_batch(state.encoder, feats)
            w_before = state.bank.weights.copy()
            # replay the dropout draw the reference makes first (trainer.py:343-348)
            rng_probe = np.random.default_rng()
            rng_probe.bit_generator.state = rng.bit_generator.state
            keep = None
            if dropout > 0:
                keep = (rng_probe.random(emb.shape) >= dropout).astype(np.float32) / np.float32(1.0 - dropout)
            rng_state = rng.bit_generator.state
            loss = trainer._batch_forward_backward(state, batch, epoch, rng, 0.0, 0.5, feats=feats)
            ids, y, origin, weights = rec["slates"]
            pre = f"s{t}_"
            out.update({
                pre + "batch_rows": batch, pre + "W_before": w_before, pre + "emb": emb,
                pre + "keep": keep if keep is not None else np.zeros((0,), np.float32),
                pre + "ids": ids, pre + "y": y, pre + "origin": origin, pre + "weights": weights,
                pre + "hard_batch": rec["hard_batch"], pre + "loss": np.float64(loss),
                pre + "grad_emb": rec["grad_emb"], pre + "uids": rec["uids"], pre + "grads": rec["grads"],
                pre + "W_after_touched": state.bank.weights[rec["uids"]].copy(), pre + "lr": np.float64(rec["lr"]),
                pre + "rng_state_seed": np.int64(seed),
            })
            # untouched-row checksum: the reference leaves them bit-identical
            mask = np.ones(L, dtype=bool)
            mask[rec["uids"]] = False
            assert np.array_equal(state.bank.weights[mask], w_before[mask])
            del rng_state
        pos_padded, n_pos = state.pos_padded, state.n_pos
        out["pos_padded"] = pos_padded
        out["n_pos"] = n_pos
    finally:
        trainer._assemble_batch_slates, trainer.encoder_backward_batch, trainer.apply_classifier_updates_arrays = orig_asm, orig_enc, orig_upd
    np.savez_compressed(os.path.join(HERE, name), **out)
    print("wrote", name)


def make_slates_fixture(name, *, L, n, B, k_p, k_h, k_r, seed, warm):
    """_assemble_batch_slates alone, including the warm phase (hard_batch None)
    and a row 0 with fewer positives than k_p (the origin quirk, :313)."""
    ds = _dataset(n, 8, L, seed, min_pos=0, max_pos=7, first_row_pos=1)
    cfg = trainer.TrainConfig(k_p=k_p, k_h=k_h, k_r=k_r, tau_s=2, tau_r=2, embed_dim=8, seed=seed, batch_size=B)
    state = trainer.TrainerState(ds, cfg)
    rng = np.random.default_rng(seed + 100)
    batch = state.active_rows[:B]
    hard = None
    epoch = 0 if warm else 3
    if not warm:
        hr = np.random.default_rng(seed + 200)
        hard = np.stack([np.sort(hr.choice(L, size=k_h, replace=False)) for _ in range(B)]).astype(np.int64)
    ids, y, origin, weights = trainer._assemble_batch_slates(state, batch, epoch, rng, hard)
    np.savez_compressed(
        os.path.join(HERE, name), L=L, k_p=k_p, k_h=k_h, k_r=k_r, rng_seed=seed + 100, batch_rows=batch,
        pos_padded=state.pos_padded, n_pos=state.n_pos, hard=hard if hard is not None else np.zeros((0, 0), np.int64),
        ids=ids, y=y, origin=origin, weights=weights, warm=warm,
    )
    print("wrote", name)


def make_refresh_fixture(name, *, L, d, N, k_h, seed, ties):
    rng = np.random.default_rng(seed)
    if ties:
        # coarse grid values and duplicated rows -> many exact score ties
        W = (rng.integers(-2, 3, size=(L, d)) / 4.0).astype(np.float32)
        W[L // 2 :] = W[: L - L // 2]
        E = (rng.integers(-1, 2, size=(N, d)) / 2.0).astype(np.float32)
        E[:3] = 0.0  # all-zero queries: every score ties (lowest ids win)
    else:
        W = rng.uniform(-1 / np.sqrt(d), 1 / np.sqrt(d), size=(L, d)).astype(np.float32)
        E = rng.standard_normal((N, d)).astype(np.float32)
    positives = [np.sort(rng.choice(L, size=int(rng.integers(0, 6)), replace=False)).astype(np.int32) for _ in range(N)]
    cache = anns.retrieve_hard_negatives(anns.build_exact(W, snapshot_epoch=4), E, positives, k_h)
    indptr, pids = _csr(positives)
    np.savez_compressed(os.path.join(HERE, name), W=W, E=E, pos_indptr=indptr, pos_ids=pids, k_h=k_h,
                        ids=cache.ids, built_from_epoch=cache.built_from_epoch)
    print("wrote", name)


def make_update_fixture(name, *, L, d, U, seed):
    rng = np.random.default_rng(seed)
    bank = classifiers.init_classifiers(L, d, "uniform-scaled", seed)
    before = bank.weights.copy()
    ids = np.sort(rng.choice(L, size=U, replace=False)).astype(np.int64)
    grads = rng.standard_normal((U, d)).astype(np.float32)
    classifiers.apply_classifier_updates_arrays(bank, ids, grads, 0.3, 1e-2)
    np.savez_compressed(os.path.join(HERE, name), W_before=before, ids=ids, grads=grads, lr=0.3, wd=1e-2, W_after=bank.weights)
    print("wrote", name)


from golden_train_spec import TRAIN_CONFIG, TRAIN_SPEC  # noqa: E402


def train_inputs(xcmix_dataset, xcmix_trainer):
    """The planted dataset, eval split and config of the train() golden (also
    rebuilt by tests/test_dropin_train_golden.py from the installed reference)."""
    sp_ = TRAIN_SPEC
    train, ev = xcmix_dataset.generate_synthetic(sp_["n_points"], sp_["n_features"], sp_["n_labels"],
                                                 sp_["labels_per_point"], noise_level=sp_["noise_level"],
                                                 seed=sp_["seed"])
    return train, ev, xcmix_trainer.TrainConfig(**TRAIN_CONFIG)


def make_train_fixture(name):
    """A whole reference train() run: the refresh pipeline (snapshot at the end
    of epoch c-2, consumed at c), Mixture slates, the sampled step, the
    encoder's Adam, the per-epoch probe and P@k (trainer.py:493-556)."""
    import xcmix.dataset as xd

    train_ds, ev, cfg = train_inputs(xd, trainer)
    enc, bank, log = trainer.train(train_ds, cfg, eval_dataset=ev)
    rec = log.records
    np.savez_compressed(
        os.path.join(HERE, name),
        loss=np.array([r.mean_slate_loss for r in rec]), probe=np.array([r.probe_full_loss for r in rec]),
        p1=np.array([np.nan if r.p_at_1 is None else r.p_at_1 for r in rec]),
        p5=np.array([np.nan if r.p_at_5 is None else r.p_at_5 for r in rec]),
        snapshot=np.array([r.snapshot_epoch for r in rec]), W=bank.weights, projection=enc.projection,
        consume=np.array([e["epoch"] for e in log.events if e["stage"] == anns.STAGE_CONSUME]),
    )
    print("wrote", name, [round(r.mean_slate_loss, 6) for r in rec])


def main():
    make_step_fixture("step_c1_parity.npz", L=2000, d=32, n=400, B=64, k_p=3, k_h=8, k_r=16, dropout=0.0, n_steps=2, seed=3)
    make_step_fixture("step_dropout.npz", L=1500, d=64, n=200, B=48, k_p=2, k_h=6, k_r=12, dropout=0.2, n_steps=1, seed=5)
    make_slates_fixture("slates_warm.npz", L=700, n=120, B=40, k_p=4, k_h=6, k_r=10, seed=7, warm=True)
    make_slates_fixture("slates_hard.npz", L=700, n=120, B=40, k_p=4, k_h=6, k_r=10, seed=8, warm=False)
    make_refresh_fixture("refresh_random.npz", L=1500, d=32, N=300, k_h=16, seed=11, ties=False)
    make_refresh_fixture("refresh_ties.npz", L=600, d=16, N=64, k_h=10, seed=12, ties=True)
    make_update_fixture("update.npz", L=500, d=24, U=120, seed=13)
    make_train_fixture("train_run.npz")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "train":
        make_train_fixture("train_run.npz")
    else:
        sys.exit(main())
