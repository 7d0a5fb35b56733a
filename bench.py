"""Benchmark of the full ASTRA classifier step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one pass of the hot path over one batch of 9216 query rows per GPU at
the LF-AmazonTitles-1.3M shape (BASELINE.json configs[3]: L=1,305,265, d=768):
the shortlist refresh of the batch's 9216 queries against the whole label set
(bf16 tcgen05 GEMM + fused top-k + fp32 re-rank, k_h=64; the reference refreshes
all N rows in one batched call, anns.py:253) and the training of the same rows
as 9 SGD minibatches of B=1024: Philox slates (k_p=8, k_h=64, k_r=512 -> S=584)
+ fused sampled-BCE fwd/bwd + SGD update of the fp32 W. This is the composite
"train samples/s (shortlist+loss+update)" with every training row refreshed
once per epoch (tau_r = 1, the most refresh-heavy schedule); refresh-only MIPS
q/s and step-only samples/s are reported beside it. Multi-GPU: W label-sharded,
per-GPU batch fixed (weak scaling), NCCL all-gather / reduce-scatter as in
paper_2409_20156_b200/shard.py.

--impl reference times the reference's own CPU path — the unmodified xcmix
package installed in baseline/_ref (anns.retrieve_hard_negatives +
trainer._batch_forward_backward) — on the host cores with the same metric, one
real step = refresh + training of one B=1024 minibatch (nothing extrapolated).

Other lines (not the driver's): --config c5shard (one 15M-label shard of the
120M config, bf16 W + Adam) and --config fullloss (the all-negatives arm at
the reference's 50K-label cap). The JSON line's `roofline` is the refresh
GEMM pass (tensor-bound), `roofline_step` the minibatch step with the
per-kernel DRAM rate of the single label-major pass (or of the two step
kernels under the deterministic schedule), `refresh_verify_ms` the refresh's
exact-fallback time (~0 when every query is proven exact).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# C4 = LF-AmazonTitles-1.3M shape, slate from SURVEY.md §8
CFG = dict(workload="LF-AmazonTitles-1.3M shape, synthetic", L=1_305_265, d=768, N=2_248_619, B=1024,
           minibatches=9, k_p=8, k_h=64, k_r=512, labels_per_point=38, tau_r=1, lr=0.05, wd=1e-4)
METRIC = "ASTRA train samples/s (shortlist+loss+update)"
UNIT = "samples/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def bench_config(world: int) -> dict:
    """The workload description shared by both arms' JSON lines."""
    c = CFG
    R = c["B"] * c["minibatches"]
    return {"workload": c["workload"], "n_labels": c["L"], "dim": c["d"], "rows_per_step_per_gpu": R,
            "minibatch": c["B"], "minibatches_per_step": c["minibatches"], "global_batch": c["B"] * world,
            "k_p": c["k_p"], "k_h": c["k_h"], "k_r": c["k_r"], "slate": c["k_p"] + c["k_h"] + c["k_r"],
            "labels_per_point": c["labels_per_point"], "tau_r": c["tau_r"], "refresh_chunk": R * world,
            "refresh_mode": "bf16_rerank", "optimizer": "sgd+wd", "parallelism": f"label-shard{world}",
            "l2": "inputs larger than L2 (W fp32 4.0 GB + snapshots 6 GB)"}


def _ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of each timed
    kernel, from the committed `ncu --set full` summary (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return {k: v["dram_bytes_per_launch"] for k, v in json.load(open(p)).items() if not k.startswith("_")}
    except (OSError, ValueError, KeyError):
        return {}


# ------------------------------------------------------------------ data
def make_batches(rng, n_batches, B, L, lpp, N, slot, n_slots):
    """Synthetic minibatches: global row ids, positives (labels_per_point
    distinct uniform labels per row, sorted), embeddings N(0,1) fp32."""
    out = []
    for t in range(n_batches):
        rows = ((slot * n_batches + t) * B + np.arange(B, dtype=np.int64)) % N
        pos = np.sort(rng.integers(0, L, size=(B, lpp)), axis=1)
        # distinct per row: collisions are rare at L=1.3M; drop duplicates
        indptr = np.zeros(B + 1, np.int64)
        flat = []
        for b in range(B):
            u = np.unique(pos[b])
            flat.append(u)
            indptr[b + 1] = indptr[b] + len(u)
        ids = np.concatenate(flat).astype(np.int32)
        emb = rng.standard_normal((B, CFG["d"]), dtype=np.float32)
        out.append(dict(rows=rows, indptr=indptr, pos=ids, emb=emb))
    return out


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2409_20156_b200 import _lib, ops
    from paper_2409_20156_b200.engine import ClassifierEngine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L, d, B, M = CFG["L"], CFG["d"], CFG["B"], CFG["minibatches"]
    k_p, k_h, k_r = CFG["k_p"], CFG["k_h"], CFG["k_r"]
    S = k_p + k_h + k_r
    R = B * M  # rows per step per GPU (refresh chunk)
    hbm, tf_burst, tf_sus, peak_kind = peaks()

    eng = ClassifierEngine(L, d, k_p=k_p, k_h=k_h, k_r=k_r, seed=0, refresh_mode="bf16_rerank")
    eng.snapshot(epoch=0)
    L_loc = eng.hi - eng.lo
    rng = np.random.default_rng(1000 + rank)
    n_steps = args.warmup + args.steps
    # host data: per step M minibatches (rows, positives CSR, embeddings)
    host = [make_batches(rng, M, B, L, CFG["labels_per_point"], CFG["N"], rank + t * world, world * n_steps)
            for t in range(n_steps)]
    dev = []
    for mbs in host:
        mb_dev = [{k: torch.from_numpy(v).cuda() for k, v in hb.items()} for hb in mbs]
        ip = np.concatenate([[0]] + [hb["indptr"][1:] + sum(int(x["indptr"][-1]) for x in mbs[:i])
                                     for i, hb in enumerate(mbs)]).astype(np.int64)
        chunk = {"emb": torch.from_numpy(np.concatenate([hb["emb"] for hb in mbs])).cuda(),
                 "indptr": torch.from_numpy(ip).cuda(),
                 "pos": torch.from_numpy(np.concatenate([hb["pos"] for hb in mbs])).cuda()}
        dev.append({"mbs": mb_dev, "chunk": chunk})
    # the stale hard-negative cache rows of each minibatch: one refresh per chunk up front
    for st in dev:
        hard, _ = eng.refresh(st["chunk"]["emb"], st["chunk"]["indptr"], st["chunk"]["pos"], k_h)
        for i, m in enumerate(st["mbs"]):
            m["hard"] = hard[i * B : (i + 1) * B].contiguous()
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * M + 2)] for _ in range(n_steps)]
    ids_keep = []

    # the refresh of the step's rows runs on a side stream concurrently with the
    # training minibatches (its output is the NEXT epoch's stale cache, as the
    # reference's background _RefreshJob thread, trainer.py:198-214), confined
    # to an SM budget so the HBM-bound step keeps the remaining SMs
    overlap = args.refresh_sms > 0
    rstream = torch.cuda.Stream() if overlap else stream
    if overlap:
        _lib.set_refresh_sm_budget(args.refresh_sms)

    def one(t, timed):
        st, e = dev[t], ev[t]
        e[0].record(stream)
        rstream.wait_stream(stream)
        with torch.cuda.stream(rstream):
            eng.refresh(st["chunk"]["emb"], st["chunk"]["indptr"], st["chunk"]["pos"], k_h)
            e[1].record(rstream)
        for i, m in enumerate(st["mbs"]):
            slates = eng.sample(m["rows"], m["indptr"], m["pos"], m["hard"], epoch=1, step=t * M + i)
            e[2 + 2 * i].record(stream)
            loss, grad_emb, status = eng.step(m["emb"], slates, CFG["lr"], CFG["wd"])
            e[3 + 2 * i].record(stream)
            if timed and i == 0:
                ids_keep.append(slates[0])
        stream.wait_stream(rstream)
        return loss, status

    # clock samples cover warm-up + timed region (the timed region alone can be
    # shorter than nvidia-smi's sampling period)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(1.0)
    for t in range(args.warmup):
        one(t, False)
    torch.cuda.synchronize()
    eng.comm.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    for name in ("refresh_gemm", "refresh_verify", "step_single", "slot_forward", "label_update"):
        _lib.kernel_timing(name)  # drop warm-up records
    _lib.kernel_timing_enable(True)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for t in range(args.warmup, n_steps):
        loss, status = one(t, True)
    t_end.record(stream)
    torch.cuda.synchronize()
    eng.comm.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    _lib.kernel_timing_enable(False)
    kt = {name: _lib.kernel_timing(name) for name in ("refresh_gemm", "refresh_verify", "step_single", "slot_forward", "label_update")}
    ops.raise_for_step_status(status)
    ms_t = torch.tensor([t_start.elapsed_time(t_end)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_total = float(ms_t.item())
    K = args.steps
    ph = {"refresh": 0.0, "sample": 0.0, "step": 0.0}
    for t in range(args.warmup, n_steps):
        e = ev[t]
        ph["refresh"] += e[0].elapsed_time(e[1])
        for i in range(M):
            ph["sample"] += (e[1 if not overlap else 0] if i == 0 else e[1 + 2 * i]).elapsed_time(e[2 + 2 * i])
            ph["step"] += e[2 + 2 * i].elapsed_time(e[3 + 2 * i])
    value = R * world * K / (ms_total / 1e3)

    # dominant kernel: the refresh GEMM pass (tcgen05 bf16 GEMM of the queries
    # against every label with the fused candidate epilogue), timed live with
    # CUDA events on its stream around each launch (astra_kernel_timing)
    q_per_refresh = R * world  # every shard scores all gathered queries
    flops = 2.0 * L_loc * d * q_per_refresh
    gemm_ms, gemm_n = kt["refresh_gemm"]
    t_gemm = gemm_ms / max(gemm_n, 1) / 1e3
    achieved_tf = flops / t_gemm / 1e12
    t_ref = ph["refresh"] / K / 1e3
    # step roofline: BASELINE.md bytes formula (U unique rows, fp32 SGD: read+write)
    U = [int(torch.unique(ids[(ids >= eng.lo) & (ids < eng.hi)]).numel()) for ids in ids_keep]
    U_mean = sum(U) / len(U)
    step_bytes = U_mean * d * (2 * 4) + 2 * B * world * d * 4 + B * world * S * 5
    t_step = ph["step"] / (K * M) / 1e3
    t_samp = ph["sample"] / (K * M) / 1e3
    step_gbs = step_bytes / t_step / 1e9
    # per-kernel HBM rates of the step (algorithmic bytes per launch / live event time)
    sgl_ms, sgl_n = kt["step_single"]
    fwd_ms, fwd_n = kt["slot_forward"]
    upd_ms, upd_n = kt["label_update"]
    fwd_bytes = B * world * S * d * 4 + B * world * d * 4 * 2  # gathered rows + emb + grad_emb
    upd_bytes = U_mean * d * 4 * 2  # each touched row read + written once (emb rows come from L2)
    traffic = _ncu_traffic()
    rate = lambda nbytes, ms_, n_: round(nbytes / (ms_ / max(n_, 1) / 1e3) / 1e9, 1)  # noqa: E731
    if sgl_n:  # the single label-major pass (default); the two-kernel launches are no-ops
        step_kernel_desc = "minibatch step (counting sort + single label-major pass: scores, loss, grad_emb, SGD row update)"
        step_kernels = {"step_single": {"launch_ms": round(sgl_ms / sgl_n, 4), "achieved_gbs": rate(upd_bytes, sgl_ms, sgl_n),
                                        "algorithmic_bytes": int(upd_bytes), "traffic": traffic.get("step_single")}}
    else:
        step_kernel_desc = "minibatch step (gather/loss/grad + counting sort + fused SGD row update)"
        step_kernels = {
            "slot_forward": {"launch_ms": round(fwd_ms / max(fwd_n, 1), 4), "achieved_gbs": rate(fwd_bytes, fwd_ms, fwd_n),
                             "algorithmic_bytes": int(fwd_bytes), "traffic": traffic.get("slot_forward")},
            "label_update": {"launch_ms": round(upd_ms / max(upd_n, 1), 4), "achieved_gbs": rate(upd_bytes, upd_ms, upd_n),
                             "algorithmic_bytes": int(upd_bytes), "traffic": traffic.get("label_update")}}
    # end-to-end: the public API with HOST buffers (pinned), copies inside the timed region
    pinned = []
    for t in range(n_steps):
        mbs = [{k: torch.from_numpy(v).pin_memory() for k, v in hb.items()} for hb in host[t]]
        for m, md in zip(mbs, dev[t]["mbs"]):
            m["hard"] = md["hard"].cpu().pin_memory()
        ch = {k: v.cpu().pin_memory() for k, v in dev[t]["chunk"].items()}
        pinned.append({"mbs": mbs, "chunk": ch})
    outs = [None] * M
    rout = None

    def one_host(t):
        nonlocal rout
        p = pinned[t]
        rstream.wait_stream(stream)
        with torch.cuda.stream(rstream):
            rout = eng.refresh_host(p["chunk"]["emb"], p["chunk"]["indptr"], p["chunk"]["pos"], k_h, out=rout)
        for i, m in enumerate(p["mbs"]):
            outs[i], _ = eng.train_step_host(m["emb"], m["rows"], m["indptr"], m["pos"], m["hard"], 1, t * M + i,
                                             CFG["lr"], CFG["wd"], out=outs[i])
        stream.wait_stream(rstream)
        eng.wait_host_outputs()  # the step's D2H results are complete when the step ends

    for t in range(args.warmup):
        one_host(t)
    torch.cuda.synchronize()
    eng.comm.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(args.warmup, n_steps):
        one_host(t)
    e1.record(stream)
    torch.cuda.synchronize()
    nbytes = lambda ts: sum(x.numel() * x.element_size() for x in ts)  # noqa: E731
    p = pinned[-1]
    h2d = nbytes(p["chunk"].values()) + sum(nbytes((m["emb"], m["rows"], m["indptr"], m["pos"], m["hard"])) for m in p["mbs"])
    d2h = nbytes([rout]) + sum(nbytes(o) for o in outs)
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = R * world * K / (float(e2e_ms.item()) / 1e3)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": round(ms_total / K, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32 W/step, bf16 tensor-core refresh + fp32 re-rank", "data": "synthetic",
        "config": dict(bench_config(world), refresh_overlap=overlap,
                       refresh_sms=args.refresh_sms if overlap else None),
        "phases_ms_per_step": {k: round(v / K, 4) for k, v in ph.items()},
        "refresh_mips_qps": round(q_per_refresh / t_ref, 1),
        # the exact fallback of the two-pass refresh (running top-k for query
        # tiles holding a flagged query): ~0 when every query was proven exact
        "refresh_verify_ms": round(kt["refresh_verify"][0] / max(kt["refresh_verify"][1], 1), 4),
        "step_only_samples_per_s": round(B * world / (t_step + t_samp), 1),
        "composite_tau_r5_samples_per_s": round(R * world / (M * (t_step + t_samp) + t_ref / 5), 1),
        "roofline": {"bound": "tensor", "kernel": "refresh_tc_kernel threshold pass (tcgen05 bf16 GEMM + fused candidate epilogue)",
                     "achieved": round(achieved_tf, 2), "peak": tf_sus, "unit": "TFLOP/s",
                     "frac": round(achieved_tf / tf_sus, 4), "traffic": traffic.get("refresh_gemm"),
                     "frac_of_burst_peak": round(achieved_tf / tf_burst, 4),
                     "algorithmic": f"2*L_shard*d*Q = {flops:.3e} flop per launch (Q={q_per_refresh})",
                     "launch_ms": round(t_gemm * 1e3, 4), "launches": gemm_n,
                     "share_of_refresh": round(t_gemm / t_ref, 4),
                     "peak_kind": f"{peak_kind} sustained bf16 (kernel timed inside a long step)"},
        "roofline_step": {"bound": "hbm", "kernel": step_kernel_desc,
                          "achieved": round(step_gbs, 1), "peak": hbm, "unit": "GB/s", "frac": round(step_gbs / hbm, 4),
                          "algorithmic": f"U*d*8 + 2*B*d*4 + B*S*5 = {step_bytes:.3e} B (U={U_mean:.0f})",
                          "peak_kind": peak_kind,
                          "kernels": step_kernels},
        "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ C5 shard emulation
C5 = dict(workload="120M-label synthetic, rank-0 shard of 8 (15M labels) emulated on one GPU", L_total=120_000_000,
          world=8, d=768, B_global=4096, k_p=16, k_h=200, k_i=200, n_cand=400, k_r=2000, labels_per_point=10,
          lr=1e-3, wd=0.0)


def run_c5shard(args):
    """BASELINE.json configs[4] as one of its 8 label shards: W (15M x 768 bf16)
    + Adam m, v (fp32) resident on this GPU; each step = the refresh of the
    global batch's 4096 queries against the shard (bf16 tcgen05 two-pass +
    bf16-row re-rank, k_h=200) + Philox slates over all 120M labels (k_p=16,
    k_h=200, k_i=200 importance, k_r=2000 -> S=2416) + the fused loss/update of
    the slots this shard owns (~1/8). The collectives of the 8-GPU job (query /
    embedding all-gathers, key all-gather, grad_emb reduce-scatter: ~40 MB per
    step over NVLink) are not run; the line reports the shard's compute time."""
    import torch

    from paper_2409_20156_b200 import _lib, ops

    torch.cuda.set_device(0)
    c = C5
    L = c["L_total"] // c["world"]
    d, B = c["d"], c["B_global"]
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    W = torch.empty((L, d), dtype=torch.bfloat16, device="cuda")
    for lo in range(0, L, 1 << 20):  # chunked init (uniform(-1/sqrt(d), 1/sqrt(d)), classifiers.py:37-40)
        hi = min(L, lo + (1 << 20))
        W[lo:hi] = ((torch.rand((hi - lo, d), device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
    m = torch.zeros((L, d), dtype=torch.float32, device="cuda")
    v = torch.zeros_like(m)
    w_absmax = W.abs().max().float().reshape(1)  # running max|W| bound (kept by the step kernels)
    snap = W.clone()
    n_steps = args.warmup + args.steps
    data = []
    for t in range(n_steps):
        rows = torch.arange(t * B, (t + 1) * B, dtype=torch.int64, device="cuda")
        pos = torch.randint(0, c["L_total"], (B, c["labels_per_point"]), device="cuda", generator=g).sort(1).values
        ip = torch.arange(0, B * c["labels_per_point"] + 1, c["labels_per_point"], dtype=torch.int64, device="cuda")
        pid = pos.to(torch.int32).reshape(-1).contiguous()
        emb = torch.randn((B, d), device="cuda", generator=g)
        hard = torch.randint(0, c["L_total"], (B, c["k_h"]), device="cuda", generator=g).to(torch.int32)
        cand = torch.randint(0, c["L_total"], (B, c["n_cand"]), device="cuda", generator=g).to(torch.int32)
        cand_q = torch.full((B, c["n_cand"]), 1.0 / c["n_cand"], device="cuda")
        data.append((rows, ip, pid, emb, hard, cand, cand_q))
    stream = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_steps)]

    def one(t):
        rows, ip, pid, emb, hard, cand, cand_q = data[t]
        e = ev[t]
        e[0].record(stream)
        ops.refresh_topk(emb, ip, pid, c["k_h"], "bf16_rerank", labels_bf16=snap)
        e[1].record(stream)
        sl = ops.sample_slates(0, 1, t, rows, ip, pid, hard, c["k_h"], c["L_total"], c["k_p"], c["k_r"], cand=cand,
                               cand_q=cand_q, k_i=c["k_i"])
        e[2].record(stream)
        res = ops.slate_step(emb, *sl, W, c["lr"], c["wd"], optimizer="adam", adam_m=m, adam_v=v, adam_step=t + 1,
                             label_offset=0, w_absmax=w_absmax)
        e[3].record(stream)
        return res, sl

    for t in range(args.warmup):
        one(t)
    torch.cuda.synchronize()
    for name in ("refresh_gemm", "refresh_verify", "step_single", "slot_forward", "label_update"):
        _lib.kernel_timing(name)
    _lib.kernel_timing_enable(True)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for t in range(args.warmup, n_steps):
        res, sl = one(t)
    t1.record(stream)
    torch.cuda.synchronize()
    _lib.kernel_timing_enable(False)
    kt = {name: _lib.kernel_timing(name) for name in ("refresh_gemm", "refresh_verify", "step_single", "slot_forward", "label_update")}
    ops.raise_for_step_status(res.status)
    K = args.steps
    ms = t0.elapsed_time(t1) / K
    ph = {"refresh": 0.0, "sample": 0.0, "step": 0.0}
    for t in range(args.warmup, n_steps):
        e = ev[t]
        ph["refresh"] += e[0].elapsed_time(e[1]) / K
        ph["sample"] += e[1].elapsed_time(e[2]) / K
        ph["step"] += e[2].elapsed_time(e[3]) / K
    ids = sl[0]
    own = ids[(ids >= 0) & (ids < L)]
    U = int(torch.unique(own).numel())
    _, tf_burst, tf_sus, peak_kind = peaks()[0], peaks()[1], peaks()[2], peaks()[3]
    hbm = peaks()[0]
    gemm_ms, gemm_n = kt["refresh_gemm"]
    flops = 2.0 * L * d * B
    achieved = flops / (gemm_ms / max(gemm_n, 1) / 1e3) / 1e12
    step_bytes = U * d * (2 * 2 + 2 * 8) + 2 * B * d * 4 + B * sl[0].shape[1] * 5
    line = {
        "metric": METRIC + " [C5 shard emulation]", "value": round(B / (ms / 1e3), 1), "unit": UNIT, "n_gpus": 1,
        "emulates_n_gpus": c["world"], "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16 W + fp32 Adam state; bf16 tcgen05 refresh + re-rank on the bf16 rows", "data": "synthetic",
        "config": {"workload": c["workload"], "n_labels_total": c["L_total"], "labels_shard": L, "dim": d,
                   "global_batch": B, "k_p": c["k_p"], "k_h": c["k_h"], "k_i": c["k_i"], "k_r": c["k_r"],
                   "slate": int(sl[0].shape[1]), "tau_r": 1, "optimizer": "adam", "owned_slots": int(own.numel()),
                   "unique_rows": U},
        "phases_ms_per_step": {k: round(v, 3) for k, v in ph.items()},
        "refresh_mips_qps_shard": round(B / (ph["refresh"] / 1e3), 1),
        "refresh_verify_ms": round(kt["refresh_verify"][0] / max(kt["refresh_verify"][1], 1), 4),
        "composite_tau_r5_samples_per_s": round(B / ((ph["sample"] + ph["step"] + ph["refresh"] / 5) / 1e3), 1),
        "roofline": {"bound": "tensor", "kernel": "refresh_tc_kernel threshold pass", "achieved": round(achieved, 2),
                     "peak": tf_sus, "unit": "TFLOP/s", "frac": round(achieved / tf_sus, 4),
                     "launch_ms": round(gemm_ms / max(gemm_n, 1), 3)},
        "roofline_step": {"bound": "hbm", "achieved": round(step_bytes / (ph["step"] / 1e3) / 1e9, 1), "peak": hbm,
                          "unit": "GB/s", "frac": round(step_bytes / (ph["step"] / 1e3) / 1e9 / hbm, 4),
                          "algorithmic": f"U*d*(2*2 + 2*8) + 2*B*d*4 + B*S*5 = {step_bytes:.3e} B (U={U})"},
        "memory_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ CPU arm
class ReferenceCPU:
    """The reference's own CPU path on this workload, timed on the host cores.

    Runs the UNMODIFIED reference package installed in baseline/_ref
    (`pip install --no-deps --target baseline/_ref /root/reference/pkg`, see
    DESIGN.md §9) through its public functions: per step, the shortlist
    refresh of one minibatch's rows, `xcmix.anns.retrieve_hard_negatives`
    (anns.py:233-256) against `build_exact` of the classifier bank, then
    `xcmix.trainer._batch_forward_backward` (trainer.py:336-395: slates,
    sampled loss fwd/bwd, the caller's small encoder + Adam, the SGD row
    update of W) on those rows with the fresh hard negatives, strategy
    Mixture (k_p=8, k_h=64, k_r=512). Each row is refreshed and trained once
    per step, as in the GPU arm's step; nothing is extrapolated. Without
    baseline/_ref it falls back to the bit-pinned NumPy port of the same
    functions (oracle/xcmix_port.py, kind "port")."""

    N_FEATURES = 768
    NNZ = 16

    def __init__(self, n_rows: int, seed: int = 7):
        c = CFG
        self.B, self.L, self.d = c["B"], c["L"], c["d"]
        ref = os.path.join(ROOT, "baseline", "_ref")
        self.kind = "port"
        if os.path.isdir(os.path.join(ref, "xcmix")):
            if ref not in sys.path:
                sys.path.insert(0, ref)
            try:
                import xcmix.anns  # noqa: F401
                import xcmix.trainer  # noqa: F401

                self.kind = "reference"
            except ImportError:
                self.kind = "port"
        rng = np.random.default_rng(seed)
        n_rows = max(n_rows, self.B)
        self.n_rows = n_rows
        self.positives = [np.unique(rng.integers(0, self.L, size=c["labels_per_point"])).astype(np.int32)
                          for _ in range(n_rows)]
        if self.kind == "reference":
            import scipy.sparse as sp
            from xcmix import anns
            from xcmix.dataset import SparseDataset
            from xcmix.trainer import TrainConfig, TrainerState

            cols = rng.integers(0, self.N_FEATURES, size=(n_rows, self.NNZ))
            vals = rng.standard_normal((n_rows, self.NNZ)).astype(np.float32)
            feats = sp.csr_matrix((vals.ravel(), cols.ravel(), np.arange(0, n_rows * self.NNZ + 1, self.NNZ)),
                                  shape=(n_rows, self.N_FEATURES), dtype=np.float32)
            feats.sum_duplicates()
            ds = SparseDataset(n_points=n_rows, n_features=self.N_FEATURES, n_labels=self.L, features=feats,
                               positives=self.positives)
            self.cfg = TrainConfig(epochs=1, batch_size=self.B, lr_encoder=0.01, lr_classifier=c["lr"],
                                   weight_decay_classifier=c["wd"], k_r=c["k_r"], k_h=c["k_h"], k_p=c["k_p"], tau_s=2,
                                   tau_r=1, strategy="Mixture", embed_dim=self.d, seed=0, dropout=0.0)
            self.state = TrainerState(ds, self.cfg)  # reference init: encoder, bank (uniform-scaled W), ...
            self.index = anns.build_exact(self.state.bank.weights, snapshot_epoch=0)
            self.cache_ids = np.zeros((n_rows, c["k_h"]), dtype=np.int32)
            self.state.caches.negative_cache = anns.NegativeCache(self.cache_ids, 0)
        else:
            W = rng.random((self.L, self.d), dtype=np.float32)
            W *= np.float32(2.0 / np.sqrt(self.d))
            W -= np.float32(1.0 / np.sqrt(self.d))
            self.W = W
            self.emb = rng.standard_normal((n_rows, self.d), dtype=np.float32)

    def step(self, t: int) -> tuple[float, float]:
        """One step over minibatch t (mod the rows): (refresh seconds, train seconds)."""
        nb = self.n_rows // self.B
        rows = (t % nb) * self.B + np.arange(self.B, dtype=np.int64)
        pos = [self.positives[r] for r in rows]
        if self.kind == "reference":
            from xcmix import anns
            from xcmix import trainer as xt

            t0 = time.perf_counter()
            emb = xt.embed_batch(self.state.encoder, self.state.dataset.features[rows])
            cache = anns.retrieve_hard_negatives(self.index, emb, pos, CFG["k_h"])
            self.cache_ids[rows] = cache.ids
            t1 = time.perf_counter()
            xt._batch_forward_backward(self.state, rows, 2, np.random.default_rng(1000 + t), 0.01, CFG["lr"])
            return t1 - t0, time.perf_counter() - t1
        from oracle import xcmix_port as port

        t0 = time.perf_counter()
        hard = port.retrieve_hard_negatives(self.W, self.emb[rows], pos, CFG["k_h"], chunk=self.B)
        t1 = time.perf_counter()
        pos_padded, n_pos = port.pad_positives(pos)
        ids, y, origin, weights = port.assemble_batch_slates(pos_padded, n_pos, np.arange(self.B), self.L, CFG["k_p"],
                                                             CFG["k_r"], np.random.default_rng(1000 + t),
                                                             hard.astype(np.int64))
        port.slate_step(self.W, self.emb[rows], None, ids, y, origin, weights, CFG["lr"], CFG["wd"])
        return t1 - t0, time.perf_counter() - t1

    def describe(self) -> str:
        what = ("xcmix (baseline/_ref, unmodified): anns.retrieve_hard_negatives + trainer._batch_forward_backward"
                if self.kind == "reference" else "oracle/xcmix_port.py (NumPy restatement of the same functions)")
        return (f"per step: refresh of B={self.B} rows vs L={self.L} + one training minibatch of those rows "
                f"(S={CFG['k_p'] + CFG['k_h'] + CFG['k_r']}); {what}; numpy/scipy/OpenBLAS threads="
                f"{os.environ.get('OPENBLAS_NUM_THREADS', os.environ.get('OMP_NUM_THREADS', 'all'))}")


def cpu_baseline(args):
    """Rank 0, N=1: one warm-up + one timed step of the reference CPU path
    (~15-30 s of host work) — a reported baseline beside the GPU line."""
    ref = ReferenceCPU(2 * CFG["B"])
    ref.step(0)
    t_ref, t_step = ref.step(1)
    B = CFG["B"]
    return {"value": round(B / (t_ref + t_step), 2), "unit": UNIT, "cores": os.cpu_count(), "kind": ref.kind,
            "sample": "1 step: " + ref.describe(), "refresh_s": round(t_ref, 3), "train_s": round(t_step, 3),
            "refresh_qps": round(B / t_ref, 2)}


def run_reference(args):
    """--impl reference: the reference's CPU path (ReferenceCPU) for --steps
    steps of B=1024 rows each (refresh + train), after one warm-up step (CPU
    code has no compilation or allocator warm-up beyond the first call; the
    --warmup steps of the GPU arm would add ~12 s each here)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    B = CFG["B"]
    ref = ReferenceCPU(B * (args.steps + 1))
    warm = 1
    for t in range(warm):
        ref.step(t)
    tr = ts = 0.0
    t_wall = time.perf_counter()
    for t in range(warm, warm + args.steps):
        a, b = ref.step(t)
        tr += a
        ts += b
    wall = time.perf_counter() - t_wall
    value = B * args.steps / wall
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warm, "warmup_requested": args.warmup,
            "ms_per_step": round(wall / args.steps * 1e3, 2), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32 (numpy; loss fp64)", "data": "synthetic",
            "config": dict(bench_config(world), rows_per_step_per_gpu=B, minibatches_per_step=1, refresh_chunk=B),
            "phases_ms_per_step": {"refresh": round(tr / args.steps * 1e3, 2), "train": round(ts / args.steps * 1e3, 2)},
            "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": os.cpu_count(), "kind": ref.kind,
                             "sample": ref.describe()},
            "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_fullloss(args):
    """The all-negatives arm (train_full_loss_baseline, trainer.py:563-616) at
    the reference's label cap (L = 50,000, d = 768, B = 1024, 38 positives per
    row): per step, scores E W^T, G and the float64 BCE, grad_emb = G W, and the
    dense SGD of every row (G^T E) — three fp32 cuBLAS GEMMs (TF32 off) +
    astra_dense_bce / astra_dense_sgd — next to the oracle port of the same
    NumPy arithmetic on the host cores (one minibatch). The dense comparison
    for the sampled arm."""
    import torch

    from oracle import xcmix_port as port
    from paper_2409_20156_b200 import ops

    torch.cuda.set_device(0)
    L, d, B, lpp = 50_000, 768, 1024, 38
    rng = np.random.default_rng(0)
    W = rng.uniform(-1 / np.sqrt(d), 1 / np.sqrt(d), size=(L, d)).astype(np.float32)
    embs = [rng.standard_normal((B, d)).astype(np.float32) for _ in range(4)]
    lists = [[np.unique(rng.integers(0, L, lpp)) for _ in range(B)] for _ in range(4)]
    csr = []
    for ls in lists:
        ip = np.zeros(B + 1, np.int64)
        np.cumsum([len(p) for p in ls], out=ip[1:])
        csr.append((torch.from_numpy(ip).cuda(), torch.from_numpy(np.concatenate(ls).astype(np.int32)).cuda()))
    Wd = torch.from_numpy(W).cuda()
    ed = [torch.from_numpy(e).cuda() for e in embs]
    stream = torch.cuda.current_stream()

    def one(t):
        e = ed[t % 4]
        loss, G, grad_emb = ops.full_loss_forward(e, Wd, *csr[t % 4])
        ops.full_loss_update(Wd, G, e, 0.01, 1e-4)
        return loss

    for t in range(args.warmup):
        one(t)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for t in range(args.steps):
        loss = one(t)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    flops = 3 * 2.0 * B * L * d
    t0 = time.perf_counter()
    Wc = W.copy()
    yb = port.dense_y(lists[0], L)
    _, G, _ = port.full_loss_forward(Wc, embs[0], None, yb)
    port.full_loss_update(Wc, G, embs[0], 0.01, 1e-4)
    t_cpu = time.perf_counter() - t0
    line = {
        "metric": "full-loss (all-negatives) arm train samples/s", "value": round(B / (ms / 1e3), 1),
        "unit": "samples/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32 (cuBLAS sgemm, TF32 off) + float64 loss", "data": "synthetic",
        "config": {"workload": "train_full_loss_baseline at the reference's label cap", "n_labels": L, "dim": d,
                   "minibatch": B, "labels_per_point": lpp},
        "roofline": {"bound": "fp32 SIMT GEMM", "achieved": round(flops / (ms / 1e3) / 1e12, 2), "unit": "TFLOP/s",
                     "algorithmic": f"3 GEMMs x 2*B*L*d = {flops:.3e} flop per step"},
        "cpu_baseline": {"value": round(B / t_cpu, 2), "unit": "samples/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": "one minibatch of the NumPy arm (oracle port), threads=all"},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c4", choices=["c4", "c5shard", "fullloss"],
                    help="c4 (default, the headline line), c5shard (120M-label config, one of 8 shards) or "
                         "fullloss (the all-negatives arm at the reference's 50K-label cap)")
    ap.add_argument("--refresh-sms", type=int, default=0,
                    help="SM budget of the refresh running concurrently with training on a side stream (0 = serial)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c5shard":
        run_c5shard(args)
    elif args.config == "fullloss":
        run_fullloss(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
