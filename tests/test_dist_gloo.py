"""Label-sharded engine over torch.distributed (gloo, world_size 2) on CPU.

The per-shard device ops run on the oracle backend (tests/oracle_backend.py);
what is under test is the multi-GPU host logic of shard.py / engine.py:
shard ranges, all-gathers of queries / positives / slates / embeddings, the
exact merge of partial top-k lists, reduce-scatter of grad_emb and the
all-reduce of the loss. Expected: refresh ids and every W shard identical to
a single-process run; grad_emb and loss equal up to summation order.
"""

import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

L, D, B, K_P, K_H, K_R = 997, 24, 16, 3, 6, 20


def _data(seed=0):
    rng = np.random.default_rng(seed)
    W = rng.uniform(-0.2, 0.2, size=(L, D)).astype(np.float32)
    world_rows = {}
    for r in range(2):
        emb = rng.standard_normal((B, D)).astype(np.float32)
        pos = [np.sort(rng.choice(L, size=int(rng.integers(1, 5)), replace=False)).astype(np.int32) for _ in range(B)]
        rows = np.arange(B, dtype=np.int64) + 1000 * r
        world_rows[r] = (emb, pos, rows)
    return W, world_rows


def _csr(pos):
    ip = np.zeros(len(pos) + 1, np.int64)
    ip[1:] = np.cumsum([len(p) for p in pos])
    return ip, np.concatenate(pos).astype(np.int32)


def _worker(rank, world, port, out_dir):
    sys.path[:0] = [ROOT, HERE]
    import oracle_backend
    from paper_2409_20156_b200.engine import ClassifierEngine

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, data = _data()
    eng = ClassifierEngine(L, D, k_p=K_P, k_h=K_H, k_r=K_R, weights=W, refresh_mode="fp32", seed=5, device="cpu",
                           backend=oracle_backend)
    eng.snapshot(0)
    emb, pos, rows = data[rank]
    ip, pid = _csr(pos)
    ids, _ = eng.refresh(torch.from_numpy(emb), torch.from_numpy(ip), torch.from_numpy(pid), K_H)
    slates = eng.sample(torch.from_numpy(rows), torch.from_numpy(ip), torch.from_numpy(pid), ids, epoch=2, step=3)
    loss, grad_emb, status = eng.step(torch.from_numpy(emb), slates, 0.3, 1e-3)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=ids.numpy(), grad_emb=grad_emb.numpy(), loss=loss.numpy(),
             status=status.numpy(), W=eng.W.numpy(), lo=eng.lo, hi=eng.hi, slate_ids=slates[0].numpy())
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_label_sharding_matches_single_process():
    sys.path[:0] = [HERE]
    import oracle_backend
    from oracle import c_oracle as co
    from paper_2409_20156_b200.engine import ClassifierEngine

    with tempfile.TemporaryDirectory() as tmp:
        mp.start_processes(_worker, args=(2, _free_port(), tmp), nprocs=2, join=True, start_method="spawn")
        res = [dict(np.load(os.path.join(tmp, f"r{r}.npz"))) for r in range(2)]
    W, data = _data()
    # refresh: exact global top-k for each rank's rows
    for r in range(2):
        emb, pos, _ = data[r]
        _, ref_ids, _ = co.refresh_fp32(emb, W, *_csr(pos), K_H)
        np.testing.assert_array_equal(res[r]["ids"], ref_ids)
    # shards partition the label range
    assert res[0]["lo"] == 0 and res[0]["hi"] == res[1]["lo"] and res[1]["hi"] == L
    # single-process step on the concatenated batch with the same slates
    emb_all = np.concatenate([data[r][0] for r in range(2)])
    pos_all = data[0][1] + data[1][1]
    rows_all = np.concatenate([data[r][2] for r in range(2)])
    ip, pid = _csr(pos_all)
    hard = torch.from_numpy(np.concatenate([res[r]["ids"] for r in range(2)]))
    one = ClassifierEngine(L, D, k_p=K_P, k_h=K_H, k_r=K_R, weights=W, refresh_mode="fp32", seed=5, device="cpu",
                           backend=oracle_backend)
    slates = one.sample(torch.from_numpy(rows_all), torch.from_numpy(ip), torch.from_numpy(pid), hard, epoch=2, step=3)
    np.testing.assert_array_equal(slates[0].numpy(), res[0]["slate_ids"])
    loss, grad_emb, status = one.step(torch.from_numpy(emb_all), slates, 0.3, 1e-3)
    W1 = one.W.numpy()
    np.testing.assert_array_equal(np.concatenate([res[0]["W"], res[1]["W"]]), W1)  # bitwise: shard-local updates
    ge = np.concatenate([res[0]["grad_emb"], res[1]["grad_emb"]])
    np.testing.assert_allclose(ge, grad_emb.numpy(), rtol=1e-5, atol=1e-6 * np.abs(grad_emb.numpy()).max())
    assert abs(float(res[0]["loss"][0]) - float(loss[0])) <= 1e-9 * abs(float(loss[0]))
    assert float(res[0]["loss"][0]) == float(res[1]["loss"][0])
    assert not res[0]["status"].any() and not status.numpy().any()
