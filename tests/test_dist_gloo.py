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


def _data(seed=0, world=2):
    rng = np.random.default_rng(seed)
    W = rng.uniform(-0.2, 0.2, size=(L, D)).astype(np.float32)
    world_rows = {}
    for r in range(world):
        emb = rng.standard_normal((B, D)).astype(np.float32)
        pos = [np.sort(rng.choice(L, size=int(rng.integers(1, 5)), replace=False)).astype(np.int32) for _ in range(B)]
        rows = np.arange(B, dtype=np.int64) + 1000 * r
        world_rows[r] = (emb, pos, rows)
    return W, world_rows


def _csr(pos):
    ip = np.zeros(len(pos) + 1, np.int64)
    ip[1:] = np.cumsum([len(p) for p in pos])
    return ip, np.concatenate(pos).astype(np.int32)


def _worker(rank, world, port, out_dir, exchange="regenerate", grad_reduce="collective"):
    sys.path[:0] = [ROOT, HERE]
    import oracle_backend
    from paper_2409_20156_b200.engine import ClassifierEngine

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, data = _data(world=world)
    eng = ClassifierEngine(L, D, k_p=K_P, k_h=K_H, k_r=K_R, weights=W, refresh_mode="fp32", seed=5, device="cpu",
                           backend=oracle_backend)
    eng.slate_exchange = exchange
    eng.grad_reduce = grad_reduce
    partial = {}
    step_fn = oracle_backend.slate_step

    def recording_step(*a, **kw):  # keep this shard's partial grad_emb / loss for the check
        res = step_fn(*a, **kw)
        partial.update(grad_emb=res.grad_emb.clone().numpy(), loss=res.loss_dev.clone().numpy())
        return res

    eng.ops = type("Ops", (), {})()
    for name in dir(oracle_backend):
        if not name.startswith("__"):
            setattr(eng.ops, name, getattr(oracle_backend, name))
    eng.ops.slate_step = recording_step
    eng.snapshot(0)
    emb, pos, rows = data[rank]
    ip, pid = _csr(pos)
    ids, _ = eng.refresh(torch.from_numpy(emb), torch.from_numpy(ip), torch.from_numpy(pid), K_H)
    slates = eng.sample(torch.from_numpy(rows), torch.from_numpy(ip), torch.from_numpy(pid), ids, epoch=2, step=3)
    loss, grad_emb, status = eng.step(torch.from_numpy(emb), slates, 0.3, 1e-3)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=ids.numpy(), grad_emb=grad_emb.numpy(), loss=loss.numpy(),
             status=status.numpy(), W=eng.W.numpy(), lo=eng.lo, hi=eng.hi, slate_ids=slates[0].numpy(),
             partial_grad=partial["grad_emb"], partial_loss=partial["loss"])
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,exchange,grad_reduce", [(2, "regenerate", "collective"), (3, "regenerate", "collective"),
                                                       (2, "gather", "collective"), (2, "gather", "ordered"),
                                                       (3, "regenerate", "ordered")])
def test_label_sharding_matches_single_process(world, exchange, grad_reduce):
    sys.path[:0] = [HERE]
    import oracle_backend
    from oracle import c_oracle as co
    from paper_2409_20156_b200.engine import ClassifierEngine

    with tempfile.TemporaryDirectory() as tmp:
        mp.start_processes(_worker, args=(world, _free_port(), tmp, exchange, grad_reduce), nprocs=world, join=True,
                           start_method="spawn")
        res = [dict(np.load(os.path.join(tmp, f"r{r}.npz"))) for r in range(world)]
    W, data = _data(world=world)
    # refresh: exact global top-k for each rank's rows (all_to_all by query owner + merge)
    for r in range(world):
        emb, pos, _ = data[r]
        _, ref_ids, _ = co.refresh_fp32(emb, W, *_csr(pos), K_H)
        np.testing.assert_array_equal(res[r]["ids"], ref_ids)
    # shards partition the label range
    assert res[0]["lo"] == 0 and res[-1]["hi"] == L
    assert all(res[r]["hi"] == res[r + 1]["lo"] for r in range(world - 1))
    # single-process step on the concatenated batch with the same slates
    emb_all = np.concatenate([data[r][0] for r in range(world)])
    pos_all = sum((data[r][1] for r in range(world)), [])
    rows_all = np.concatenate([data[r][2] for r in range(world)])
    ip, pid = _csr(pos_all)
    hard = torch.from_numpy(np.concatenate([res[r]["ids"] for r in range(world)]))
    one = ClassifierEngine(L, D, k_p=K_P, k_h=K_H, k_r=K_R, weights=W, refresh_mode="fp32", seed=5, device="cpu",
                           backend=oracle_backend)
    slates = one.sample(torch.from_numpy(rows_all), torch.from_numpy(ip), torch.from_numpy(pid), hard, epoch=2, step=3)
    for r in range(world):  # every shard drew (or received) the same global slates
        np.testing.assert_array_equal(slates[0].numpy(), res[r]["slate_ids"])
    loss, grad_emb, status = one.step(torch.from_numpy(emb_all), slates, 0.3, 1e-3)
    W1 = one.W.numpy()
    np.testing.assert_array_equal(np.concatenate([res[r]["W"] for r in range(world)]), W1)  # bitwise: shard-local
    ge = np.concatenate([res[r]["grad_emb"] for r in range(world)])
    np.testing.assert_allclose(ge, grad_emb.numpy(), rtol=1e-5, atol=1e-6 * np.abs(grad_emb.numpy()).max())
    assert abs(float(res[0]["loss"][0]) - float(loss[0])) <= 1e-9 * abs(float(loss[0]))
    assert all(float(res[0]["loss"][0]) == float(res[r]["loss"][0]) for r in range(world))
    assert not res[0]["status"].any() and not status.numpy().any()
    if grad_reduce == "ordered":
        # each rank's grad_emb rows and the loss are the shards' partials summed
        # left to right in rank order (bitwise; independent of the collective)
        for r in range(world):
            acc = res[0]["partial_grad"][r * B : (r + 1) * B].copy()
            for q in range(1, world):
                acc += res[q]["partial_grad"][r * B : (r + 1) * B]
            np.testing.assert_array_equal(res[r]["grad_emb"], acc)
            lacc = res[0]["partial_loss"].copy()
            for q in range(1, world):
                lacc += res[q]["partial_loss"]
            np.testing.assert_array_equal(res[r]["loss"], lacc)


def _comm_worker(rank, world, port, out_dir):
    sys.path[:0] = [ROOT, HERE]
    from paper_2409_20156_b200.shard import Comm, gather_csr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = Comm()
    t = torch.arange(world * 4, dtype=torch.int64).view(world * 2, 2) + 1000 * rank
    ag = c.all_gather(t)
    a2a = c.all_to_all(t)
    rs = c.reduce_scatter(t.double())
    ar = c.all_reduce(torch.tensor([float(rank + 1)], dtype=torch.float64))
    ip = torch.tensor([0, rank + 1, rank + 3], dtype=torch.int64)
    ids = torch.arange(rank + 3, dtype=torch.int32) + 100 * rank
    gip, gids = gather_csr(c, ip, ids)
    np.savez(os.path.join(out_dir, f"c{rank}.npz"), ag=ag.numpy(), a2a=a2a.numpy(), rs=rs.numpy(), ar=ar.numpy(),
             gip=gip.numpy(), gids=gids.numpy())
    dist.destroy_process_group()


def test_comm_collective_semantics():
    """The tensor-form collectives shard.Comm issues (the same calls as on
    NCCL): all_gather_into_tensor, all_to_all_single, reduce_scatter_tensor,
    all_reduce, and the ragged CSR gather."""
    world = 3
    with tempfile.TemporaryDirectory() as tmp:
        mp.start_processes(_comm_worker, args=(world, _free_port(), tmp), nprocs=world, join=True, start_method="spawn")
        res = [dict(np.load(os.path.join(tmp, f"c{r}.npz"))) for r in range(world)]
    ts = [np.arange(world * 4, dtype=np.int64).reshape(world * 2, 2) + 1000 * r for r in range(world)]
    for r in range(world):
        np.testing.assert_array_equal(res[r]["ag"], np.concatenate(ts))
        np.testing.assert_array_equal(res[r]["a2a"], np.stack([t[2 * r : 2 * r + 2] for t in ts]))
        np.testing.assert_array_equal(res[r]["rs"], sum(t.astype(np.float64) for t in ts)[2 * r : 2 * r + 2])
        assert float(res[r]["ar"][0]) == sum(range(1, world + 1))
        counts = sum(([1 + q, 2] for q in range(world)), [])
        np.testing.assert_array_equal(res[r]["gip"], np.concatenate([[0], np.cumsum(counts)]))
        np.testing.assert_array_equal(res[r]["gids"], np.concatenate([np.arange(q + 3) + 100 * q for q in range(world)]))


def _rerank_worker(rank, world, port, out_dir, global_threshold, global_candidates=False):
    sys.path[:0] = [ROOT, HERE]
    import oracle_backend
    from paper_2409_20156_b200.engine import ClassifierEngine

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, data = _data(seed=4, world=world)
    eng = ClassifierEngine(L, D, k_p=K_P, k_h=K_H, k_r=K_R, weights=W, refresh_mode="bf16_rerank", seed=5,
                           device="cpu", backend=oracle_backend)
    eng.global_rerank_threshold = global_threshold
    eng.global_candidate_threshold = global_candidates
    eng.snapshot(0)
    emb, pos, _ = data[rank]
    ip, pid = _csr(pos)
    ids, scores = eng.refresh(torch.from_numpy(emb), torch.from_numpy(ip), torch.from_numpy(pid), K_H)
    np.savez(os.path.join(out_dir, f"rr{rank}.npz"), ids=ids.numpy(), scores=scores.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,global_threshold,global_candidates",
                         [(2, True, False), (3, True, False), (2, False, False), (2, True, True), (3, True, True)])
def test_sharded_bf16_rerank_matches_single_process(world, global_threshold, global_candidates):
    """BF16_RERANK over label shards (engine._refresh_sharded_rerank: shard
    bf16 top-k' -> owners merge -> global k'-th key tau -> each shard re-ranks
    only its candidates >= tau -> fp32 lists merged) returns the single-process
    BF16_RERANK result, ids and scores; so does the full per-shard re-rank."""
    sys.path[:0] = [HERE]
    import oracle_backend
    from paper_2409_20156_b200.engine import ClassifierEngine

    with tempfile.TemporaryDirectory() as tmp:
        mp.start_processes(_rerank_worker, args=(world, _free_port(), tmp, global_threshold, global_candidates),
                           nprocs=world, join=True, start_method="spawn")
        res = [dict(np.load(os.path.join(tmp, f"rr{r}.npz"))) for r in range(world)]
    W, data = _data(seed=4, world=world)
    one = ClassifierEngine(L, D, k_p=K_P, k_h=K_H, k_r=K_R, weights=W, refresh_mode="bf16_rerank", seed=5,
                           device="cpu", backend=oracle_backend)
    one.snapshot(0)
    for r in range(world):
        emb, pos, _ = data[r]
        ip, pid = _csr(pos)
        ids, scores = one.refresh(torch.from_numpy(emb), torch.from_numpy(ip), torch.from_numpy(pid), K_H)
        np.testing.assert_array_equal(res[r]["ids"], ids.numpy())
        np.testing.assert_array_equal(res[r]["scores"], scores.numpy())
