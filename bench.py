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
import gc
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
# BASELINE.json configs[0..2] (SURVEY.md §8 parameters); the default line is C4 above
CONFIGS = {
    "c4": dict(CFG),
    "c1": dict(workload="synthetic tiny XC (BASELINE configs[0]): L=10K, d=64", L=10_000, d=64, N=50_000, B=256,
               minibatches=9, k_p=4, k_h=16, k_r=16, labels_per_point=3, tau_r=1, lr=0.05, wd=1e-4),
    "c2": dict(workload="LF-AmazonTitles-131K shape, synthetic", L=131_073, d=768, N=294_805, B=1024, minibatches=9,
               k_p=8, k_h=64, k_r=512, labels_per_point=5, tau_r=1, lr=0.05, wd=1e-4),
    "c3": dict(workload="LF-WikiSeeAlso-320K shape, synthetic (refresh every epoch)", L=312_330, d=768, N=693_082,
               B=1024, minibatches=9, k_p=8, k_h=64, k_r=512, labels_per_point=5, tau_r=1, lr=0.05, wd=1e-4),
}
METRIC = "ASTRA train samples/s (shortlist+loss+update)"
REFRESH_MODE = ["bf16_rerank"]  # set from --refresh-mode
UNIT = "samples/s"


def fp8_peak(tf_burst):
    """Dense e4m3 denominator: the measured cuBLASLt figure (scripts/fp8_peak.py
    -> profiles/fp8_peak.json, measured on this pool's B200), else 2 x the
    measured bf16 burst."""
    p = os.path.join(ROOT, "profiles", "fp8_peak.json")
    if os.path.exists(p):
        return json.load(open(p))["fp8_e4m3_tflops"], "measured here (cuBLASLt e4m3 8192^3 burst, profiles/fp8_peak.json)"
    return 2.0 * tf_burst, "2 x the measured bf16 burst (no measured fp8 figure)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------------ clocks
def _ev():
    """A timing event whose CUDA event exists already (torch creates it lazily
    at the first record; creation inside a timed region can stall the host)."""
    import torch

    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


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
                 "-lms", os.environ.get("ASTRA_BENCH_SMI_MS", "20")], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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
            "refresh_mode": REFRESH_MODE[0], "optimizer": "sgd+wd", "parallelism": f"label-shard{world}",
            "l2": ("inputs larger than L2 (W fp32 + snapshots >= 3 x L*d*4 B)" if c["L"] * c["d"] * 12 >= 256 * 2**20
                   else "L2 flushed between timed steps (512 MB write outside the per-step events)")}


def _ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of each timed
    kernel, from the committed `ncu --set full` summary (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return {k: v["dram_bytes_per_launch"] for k, v in json.load(open(p)).items() if not k.startswith("_")}
    except (OSError, ValueError, KeyError):
        return {}


# ------------------------------------------------------------------ data
def clustered_centers(d, n_clusters=2000, seed=5):
    """Cluster centres of the trained-like W of --w-init clustered (unit-variance
    coordinates / sqrt(d)) and their Zipf popularity."""
    rng = np.random.default_rng(seed)
    centers = (rng.standard_normal((n_clusters, d)) / np.sqrt(d)).astype(np.float32)
    pop = 1.0 / np.arange(1, n_clusters + 1, dtype=np.float64) ** 1.1
    return centers, pop / pop.sum()


def clustered_w(L, d, centers, pop, seed, dup_frac=0.02):
    """Trained-like W (the refresh tests' clustered heavy-tailed matrix,
    tests/test_gpu_refresh_scale.py): rows = a Zipf-popular cluster centre +
    noise, log-normal row norms, 2% of the rows copies of 16 hub rows (exact
    score ties across far-apart ids). Breaks the two-pass plan's i.i.d. score
    assumption: candidate lists overflow and queries take the verify pass."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    C = torch.from_numpy(centers).cuda()
    assign = torch.multinomial(torch.from_numpy(pop).float().cuda(), L, replacement=True, generator=g)
    W = torch.empty((L, d), device="cuda")
    for lo in range(0, L, 1 << 18):
        hi = min(L, lo + (1 << 18))
        noise = torch.randn((hi - lo, d), device="cuda", generator=g) * (0.35 / d ** 0.5)
        scale = torch.exp(torch.randn((hi - lo, 1), device="cuda", generator=g) * 0.5)
        W[lo:hi] = (C[assign[lo:hi]] + noise) * scale
    n_dup = int(L * dup_frac)
    hubs = torch.randint(0, L, (16,), device="cuda", generator=g)
    dst = torch.randint(0, L, (n_dup,), device="cuda", generator=g)
    W[dst] = W[hubs[torch.randint(0, 16, (n_dup,), device="cuda", generator=g)]]
    return W


def make_batches(rng, n_batches, B, L, lpp, N, slot, n_slots, centers=None):
    """Synthetic minibatches: global row ids, positives (labels_per_point
    distinct uniform labels per row, sorted), embeddings N(0,1) fp32 (with
    `centers`: a Zipf-popular cluster centre x sqrt(d) + N(0, 0.25) noise, the
    queries of the clustered W)."""
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
        if centers is None:
            emb = rng.standard_normal((B, CFG["d"]), dtype=np.float32)
        else:
            which = rng.zipf(1.3, size=B) % centers.shape[0]
            emb = (centers[which] * np.sqrt(CFG["d"]) + 0.5 * rng.standard_normal((B, CFG["d"]))).astype(np.float32)
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
        if rank == 0:
            sys.stderr.write(f"[bench] NCCL {'.'.join(map(str, torch.cuda.nccl.version()))} up: world={world} "
                             f"(--gpus {args.gpus}), device {torch.cuda.get_device_name(local)}\n")
    if world != args.gpus:
        sys.exit(f"bench.py: world size {world} != --gpus {args.gpus}")
    L, d, B, M = CFG["L"], CFG["d"], CFG["B"], CFG["minibatches"]
    k_p, k_h, k_r = CFG["k_p"], CFG["k_h"], CFG["k_r"]
    S = k_p + k_h + k_r
    R = B * M  # rows per step per GPU (refresh chunk)
    hbm, tf_burst, tf_sus, peak_kind = peaks()

    eng = ClassifierEngine(L, d, k_p=k_p, k_h=k_h, k_r=k_r, seed=0, refresh_mode=args.refresh_mode)
    centers = None
    if args.w_init == "clustered":
        centers, pop = clustered_centers(d)
        Wc = clustered_w(eng.hi - eng.lo, d, centers, pop, seed=11 + rank)
        eng.W.copy_(Wc)
        eng.w_absmax.copy_(Wc.abs().amax().reshape(1))
        del Wc
    eng.snapshot(epoch=0)
    L_loc = eng.hi - eng.lo
    rng = np.random.default_rng(1000 + rank)
    n_steps = args.warmup + args.steps
    # host data: per step M minibatches (rows, positives CSR, embeddings)
    host = [make_batches(rng, M, B, L, CFG["labels_per_point"], CFG["N"], rank + t * world, world * n_steps,
                         centers=centers)
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
    ev = [[_ev() for _ in range(2 * M + 2)] for _ in range(n_steps)]
    ids_keep = []

    # the refresh of the step's rows runs on a side stream concurrently with the
    # training minibatches (its output is the NEXT epoch's stale cache, as the
    # reference's background _RefreshJob thread, trainer.py:198-214), confined
    # to an SM budget so the HBM-bound step keeps the remaining SMs
    overlap = args.refresh_sms > 0
    rstream = torch.cuda.Stream() if overlap else stream
    if overlap:
        _lib.set_refresh_sm_budget(args.refresh_sms)

    host_ts = [] if os.environ.get("ASTRA_BENCH_PHASE_DUMP") else None

    def one(t, timed, mode=None, reuse_start=False):
        st, e = dev[t], ev[t]
        if not reuse_start:
            e[0].record(stream)
        rstream.wait_stream(stream)
        with torch.cuda.stream(rstream):
            eng.refresh(st["chunk"]["emb"], st["chunk"]["indptr"], st["chunk"]["pos"], k_h, mode=mode)
            e[1].record(rstream)
        for i, m in enumerate(st["mbs"]):
            if host_ts is not None and timed:
                host_ts.append((t, i, time.perf_counter()))
            slates = eng.sample(m["rows"], m["indptr"], m["pos"], m["hard"], epoch=1, step=t * M + i)
            e[2 + 2 * i].record(stream)
            loss, grad_emb, status = eng.step(m["emb"], slates, CFG["lr"], CFG["wd"])
            e[3 + 2 * i].record(stream)
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
    t_start = _ev()
    t_end = _ev()
    # working sets that fit in L2 (C1: W is 2.5 MB) are flushed between timed
    # steps (a 512 MB write, outside the per-step events) so every step starts cold
    flush = L_loc * d * 4 * 3 < 256 * 2**20
    flush_buf = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda") if flush else None
    ends = [_ev() for _ in range(args.warmup, n_steps)] if flush else []
    torch.cuda.synchronize()
    t_start.record(stream)
    for t in range(args.warmup, n_steps):
        if flush:
            flush_buf.fill_(t & 0xFF)
            ev[t][0].record(stream)
        loss, status = one(t, True, reuse_start=flush)
        if flush:
            ends[t - args.warmup].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    eng.comm.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    _lib.kernel_timing_enable(False)
    kt = {name: _lib.kernel_timing(name) for name in ("refresh_gemm", "refresh_verify", "step_single", "slot_forward", "label_update")}
    ops.raise_for_step_status(status)
    if flush:
        ms_steps = sum(ev[t][0].elapsed_time(ends[i]) for i, t in enumerate(range(args.warmup, n_steps)))
    else:
        ms_steps = t_start.elapsed_time(t_end)
    ms_t = torch.tensor([ms_steps], dtype=torch.float64, device="cuda")
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
    if os.environ.get("ASTRA_BENCH_PHASE_DUMP"):  # per-step sample intervals (host-stall diagnosis)
        for t in range(args.warmup, n_steps):
            e = ev[t]
            print("step", t, "sample_ms", [round((e[1] if i == 0 else e[1 + 2 * i]).elapsed_time(e[2 + 2 * i]), 3)
                                           for i in range(M)], file=sys.stderr)
        gaps = sorted(((b[2] - a_[2]) * 1e3, a_[0], a_[1]) for a_, b in zip(host_ts, host_ts[1:]))[-3:]
        print("largest host gaps between sampler calls (ms, step, minibatch):", [(round(g, 2), t_, i_) for g, t_, i_ in gaps],
              file=sys.stderr)
    value = R * world * K / (ms_total / 1e3)

    # dominant kernel: the refresh GEMM pass (tcgen05 bf16 GEMM of the queries
    # against every label with the fused candidate epilogue), timed live with
    # CUDA events on its stream around each launch (astra_kernel_timing)
    q_per_refresh = R * world  # every shard scores all gathered queries
    flops = 2.0 * L_loc * d * q_per_refresh
    gemm_ms, gemm_n = kt["refresh_gemm"]
    t_gemm = gemm_ms / max(gemm_n, 1) / 1e3
    achieved_tf = flops / t_gemm / 1e12
    if args.refresh_mode == "fp8_rerank":
        f8, peak_kind_gemm = fp8_peak(tf_burst)
        tf_sus, tf_burst = tf_sus * f8 / tf_burst, f8  # (sustained: the bf16 sustained/burst ratio)
    else:
        peak_kind_gemm = f"{peak_kind} burst bf16 (each launch is timed on its own)"
    t_ref = ph["refresh"] / K / 1e3
    # step roofline: BASELINE.md bytes formula (U unique rows, fp32 SGD: read+write)
    # (the timed steps' first-minibatch slates, redrawn here: Philox keyed by
    # (seed, epoch, step) gives the same ids; keeping them alive inside the
    # timed region made the caching allocator cudaMalloc a new segment every
    # ~8 steps, a 30-130 ms host stall, profiles/r02s3/stall_ab.txt)
    for t in range(args.warmup, n_steps):
        m = dev[t]["mbs"][0]
        ids_keep.append(eng.sample(m["rows"], m["indptr"], m["pos"], m["hard"], epoch=1, step=t * M)[0])
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
    # refresh parity at the benched shape (outside the timed region): the
    # production ids (two-pass bf16 + fp32 re-rank) of the last step's chunk
    # against the fp32-exact mode (sequential fmaf = the C oracle's arithmetic,
    # tests/test_gpu_refresh_scale.py) on every query of the chunk
    st = dev[n_steps - 1]["chunk"]
    prod_ids, _ = eng.refresh(st["emb"], st["indptr"], st["pos"], k_h)
    flagged = ops.refresh_flagged(R * world, L_loc, d, k_h, args.refresh_mode)
    exact_ids, _ = eng.refresh(st["emb"], st["indptr"], st["pos"], k_h, mode="fp32")
    same = prod_ids == exact_ids
    hits = (prod_ids.unsqueeze(2) == exact_ids.unsqueeze(1)).any(2).sum(1).double() / k_h
    refresh_parity = {"vs": "fp32-exact mode (= C oracle arithmetic)", "queries": int(prod_ids.shape[0]),
                      "recall_at_k": round(float(hits.mean()), 6), "rows_bit_exact": round(float(same.all(1).double().mean()), 6),
                      "flagged_for_verify": int(flagged)}
    # the same job with the e4m3 candidate pass (kind::f8f6f4, twice the
    # tensor rate; fp32-exact re-rank of k' = 2k candidates): an extension
    # beside the north star's bf16 line, with its own parity on the same chunk
    alt_fp8 = None
    if not args.no_alt_fp8 and args.refresh_mode != "fp8_rerank" and d % 128 == 0 and eng.snap_f32 is not None:
        eng.snap_f8 = ops.quantize_e4m3(eng.snap_f32)
        for t in range(min(2, args.warmup)):
            one(t, False, mode="fp8_rerank")
        torch.cuda.synchronize()
        eng.comm.barrier()
        _lib.kernel_timing("refresh_gemm")
        _lib.kernel_timing_enable(True)
        a0, a1 = _ev(), _ev()
        a0.record(stream)
        for t in range(args.warmup, n_steps):
            one(t, False, mode="fp8_rerank")
        a1.record(stream)
        torch.cuda.synchronize()
        eng.comm.barrier()
        _lib.kernel_timing_enable(False)
        g8_ms, g8_n = _lib.kernel_timing("refresh_gemm")
        ms8 = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ms8, op=dist.ReduceOp.MAX)
        ms8 = float(ms8.item())
        r_ms = sum(ev[t][0].elapsed_time(ev[t][1]) for t in range(args.warmup, n_steps)) / K
        f8_ids, _ = eng.refresh(st["emb"], st["indptr"], st["pos"], k_h, mode="fp8_rerank")
        hits8 = (f8_ids.unsqueeze(2) == exact_ids.unsqueeze(1)).any(2).sum(1).double() / k_h
        f8_peak_tf, f8_kind = fp8_peak(tf_burst)
        ach8 = flops / (g8_ms / max(g8_n, 1) / 1e3) / 1e12
        alt_fp8 = {"refresh_mode": "fp8_rerank", "value": round(R * world * K / (ms8 / 1e3), 1), "unit": UNIT,
                   "ms_per_step": round(ms8 / K, 4), "refresh_ms_per_step": round(r_ms, 4),
                   "refresh_parity": {"recall_at_k": round(float(hits8.mean()), 6),
                                      "rows_bit_exact": round(float((f8_ids == exact_ids).all(1).double().mean()), 6)},
                   "roofline": {"bound": "tensor", "achieved": round(ach8, 2), "peak": f8_peak_tf, "unit": "TFLOP/s",
                                "frac": round(ach8 / f8_peak_tf, 4), "launch_ms": round(g8_ms / max(g8_n, 1), 4),
                                "peak_kind": f8_kind},
                   "note": "not the headline: the north star specifies the bf16 candidate pass"}
        eng.snap_f8 = None
    del exact_ids
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
    e0 = _ev()
    e1 = _ev()
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
        "dtype": f"fp32 W/step, {args.refresh_mode.split('_')[0]} tensor-core refresh + fp32 re-rank", "data": "synthetic",
        "config": dict(bench_config(world), refresh_overlap=overlap,
                       refresh_sms=args.refresh_sms if overlap else None,
                       **({"w_init": "clustered heavy-tailed W (2000 Zipf clusters, log-normal norms, 2% duplicated "
                                     "hub rows), queries near popular clusters"} if args.w_init == "clustered" else {})),
        "phases_ms_per_step": {k: round(v / K, 4) for k, v in ph.items()},
        "refresh_mips_qps": round(q_per_refresh / t_ref, 1),
        # the exact fallback of the two-pass refresh (running top-k for query
        # tiles holding a flagged query): ~0 when every query was proven exact
        "refresh_verify_ms": round(kt["refresh_verify"][0] / max(kt["refresh_verify"][1], 1), 4),
        "refresh_parity": refresh_parity,
        "alt_fp8_refresh": alt_fp8,
        "step_only_samples_per_s": round(B * world / (t_step + t_samp), 1),
        "composite_tau_r5_samples_per_s": round(R * world / (M * (t_step + t_samp) + t_ref / 5), 1),
        "roofline": {"bound": "tensor", "kernel": "refresh_tc_kernel threshold pass (tcgen05 bf16 GEMM + fused candidate epilogue)",
                     "achieved": round(achieved_tf, 2), "peak": tf_burst, "unit": "TFLOP/s",
                     "frac": round(achieved_tf / tf_burst, 4), "traffic": traffic.get("refresh_gemm"),
                     "frac_of_sustained_peak": round(achieved_tf / tf_sus, 4),
                     "algorithmic": f"2*L_shard*d*Q = {flops:.3e} flop per launch (Q={q_per_refresh})",
                     "operands": args.refresh_mode.split("_")[0],
                     "launch_ms": round(t_gemm * 1e3, 4), "launches": gemm_n,
                     "share_of_refresh": round(t_gemm / t_ref, 4),
                     "peak_kind": peak_kind_gemm},
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


# ------------------------------------------------------------------ N-GPU emulation on one GPU
def run_emulate(args):
    """Rank 0's share of an N-GPU C4 job, on one GPU (--emulate N).

    Rank r of the label-sharded job (shard.py) owns L/N labels of W and, per
    step, (a) refreshes ALL N ranks' query rows (N x 9216 after the query
    all-gather) against its shard and merges the N partial lists of its own
    rows (after the key all-to-all), then (b) per minibatch draws the slates
    of all N x 1024 rows (Philox over the global label range, identical on
    every rank) and runs the fused loss/update for the slots it owns (~1/N).
    This runs exactly that compute on one GPU, with synthetic stand-ins for
    the other ranks' rows; the collectives are NOT run and their bytes per
    rank are reported (collective_bytes_per_rank_per_step), so the per-rank
    compute cost of the N = 2/4/8 configurations is measured on one B200.
    value = N x 9216 rows / per-rank step time = the whole job's throughput
    if the collectives were free and the ranks in lockstep (an upper bound
    for the real N-GPU run, which --gpus N measures)."""
    import torch

    from paper_2409_20156_b200 import _lib, ops
    from paper_2409_20156_b200.engine import init_uniform_scaled
    from paper_2409_20156_b200.shard import shard_range

    N = args.emulate
    torch.cuda.set_device(0)
    c = CFG
    L, d, B, M = c["L"], c["d"], c["B"], c["minibatches"]
    k_p, k_h, k_r, lpp = c["k_p"], c["k_h"], c["k_r"], c["labels_per_point"]
    S = k_p + k_h + k_r
    lo, hi = shard_range(L, 0, N)
    Lr = hi - lo
    R = B * M
    Rg, Bg = R * N, B * N
    hbm, tf_burst, _, peak_kind = peaks()
    W = init_uniform_scaled(Lr, d, 1, "cuda")
    w_absmax = W.abs().amax().reshape(1).float()
    snap_f32 = W.clone()
    fp8 = args.refresh_mode == "fp8_rerank"
    snap_lp = ops.quantize_e4m3(snap_f32) if fp8 else ops.f32_to_bf16(snap_f32)
    lp = {"labels_e4m3": snap_lp} if fp8 else {"labels_bf16": snap_lp}
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    n_steps = args.warmup + args.steps
    data = []
    for t in range(n_steps):
        q = torch.randn((Rg, d), device="cuda", generator=g)
        pid = torch.randint(0, L, (Rg, lpp), device="cuda", generator=g).sort(1).values.to(torch.int32).reshape(-1)
        # distinct sorted hard ids per row (the stale cache rows of the step's rows)
        hard = (torch.randint(0, L - k_h, (Rg, k_h), device="cuda", generator=g).sort(1).values
                + torch.arange(k_h, device="cuda")).to(torch.int32)
        data.append((q, pid, hard))
    ip_step = torch.arange(0, Rg * lpp + 1, lpp, dtype=torch.int64, device="cuda")
    ip_mb = torch.arange(0, Bg * lpp + 1, lpp, dtype=torch.int64, device="cuda")
    ip_b = ip_mb[: B + 1]
    regen = args.slate_exchange == "regenerate"

    def slates_of(t, i, n_rows):
        q, pid, hard = data[t]
        rows = torch.arange((t * M + i) * Bg, (t * M + i) * Bg + n_rows, dtype=torch.int64, device="cuda")
        return ops.sample_slates(0, 1, t * M + i, rows, ip_mb[: n_rows + 1], pid[i * Bg * lpp:(i * Bg + n_rows) * lpp],
                                 hard[i * Bg:i * Bg + n_rows], k_h, L, k_p, k_r)

    # "gather" (engine default): rank 0 samples its own B rows, the other
    # ranks' slates arrive by all-gather; their slates are drawn up front here
    full = None if regen else [[slates_of(t, i, Bg) for i in range(M)] for t in range(n_steps)]
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = [[_ev() for _ in range(3 + 2 * M)] for _ in range(n_steps)]
    keep_ids = []

    # BF16_RERANK over shards (engine._refresh_sharded_rerank): this shard's bf16
    # top-k' of all rows, the owner's merge of the N lists of its R rows (the
    # global k'-th key tau), then the fp32 re-rank of only the candidates >= tau.
    # tau needs the other shards' lists, which this single-GPU emulation does not
    # compute: it stands in this shard's ceil(k'/N)-th key (the expected share of
    # an i.i.d. shard in the global top-k'), so the re-rank does the real job's
    # expected work; the merge runs on this shard's list replicated N times.
    global_rr = args.refresh_mode == "bf16_rerank" and not args.emulate_full_rerank
    kc = ops.rerank_candidates_count(k_h)
    flip = torch.tensor(-(2 ** 63), dtype=torch.int64, device="cuda")
    # ... and the candidate pass with a global threshold (engine._candidates_global):
    # the shard's sample statistics (j largest sampled group maxima), the global
    # j-th largest (proxy: this shard's ceil(j/N)-th: the expected position of the
    # global j-th among an i.i.d. shard's samples), the local candidates at or
    # above it, the verify set (proxy: this shard's count x N < k' or overflow)
    j_sh = ops.refresh_plan_j(Rg, Lr, d, kc) if global_rr and not args.emulate_shard_candidates else 0

    def one(t, timed):
        q, pid, hard = data[t]
        e = ev[t]
        e[0].record(stream)
        if global_rr and j_sh > 0:
            top = ops.refresh_sharded_stage(1, q, ip_step, pid, kc, snap_lp, label_offset=lo)
            jl = -(-j_sh // N)
            gtau = (top.to(torch.int64) & 0xFFFFFFFF).topk(jl, dim=1).values[:, jl - 1] << 32
            ck, cnt, ovf = ops.refresh_sharded_stage(2, q, ip_step, pid, kc, snap_lp, label_offset=lo, tau_keys=gtau)
            need = ((cnt.to(torch.int64) * N < kc) | (ovf > 0)).to(torch.int32)
            ckeys = ops.refresh_sharded_stage(3, q, ip_step, pid, kc, snap_lp, label_offset=lo, io_keys=ck,
                                              flags=need)
        if global_rr:
            if j_sh == 0:
                ckeys, _, _ = ops.refresh_topk(q, ip_step, pid, kc, "bf16", labels_f32=snap_f32, label_offset=lo,
                                               **lp)
            ops.topk_merge(ckeys[:R].unsqueeze(0).expand(N, R, kc).contiguous(), kc)  # owner's merge (stand-in data)
            tau = ckeys[:, -(-kc // N) - 1].contiguous()  # (proxy of the all-gathered global tau)
            cand = torch.where((ckeys ^ flip) >= (tau[:, None] ^ flip), ckeys, torch.zeros_like(ckeys))
            keys, _, _ = ops.rerank_candidates(q, cand, k_h, labels_f32=snap_f32, label_offset=lo)
        else:
            keys, _, _ = ops.refresh_topk(q, ip_step, pid, k_h, args.refresh_mode, labels_f32=snap_f32,
                                          label_offset=lo, **lp)
        e[1].record(stream)
        ops.topk_merge(keys.view(N, R, k_h), k_h)  # the N shards' lists of this rank's R rows
        e[2].record(stream)
        for i in range(M):
            if regen:
                sl = slates_of(t, i, Bg)
            else:
                slates_of(t, i, B)  # this rank's own rows (rows 0..B-1 of the global minibatch)
                sl = full[t][i]
            e[3 + 2 * i].record(stream)
            emb = q[i * Bg:(i + 1) * Bg]
            res = ops.slate_step(emb, *sl, W, c["lr"], c["wd"], label_offset=lo, w_absmax=w_absmax)
            e[4 + 2 * i].record(stream)
            if timed and i == 0:
                keep_ids.append(sl[0])
        return res

    for t in range(args.warmup):
        one(t, False)
    torch.cuda.synchronize()
    for name in ("refresh_gemm", "step_single"):
        _lib.kernel_timing(name)
    _lib.kernel_timing_enable(True)
    clocks = ClockSampler(0)
    clocks.start()
    t0, t1 = _ev(), _ev()
    t0.record(stream)
    for t in range(args.warmup, n_steps):
        res = one(t, True)
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    _lib.kernel_timing_enable(False)
    kt = {name: _lib.kernel_timing(name) for name in ("refresh_gemm", "step_single")}
    ops.raise_for_step_status(res.status)
    K = args.steps
    ms = t0.elapsed_time(t1) / K
    ph = {"refresh": 0.0, "merge": 0.0, "sample": 0.0, "step": 0.0}
    for t in range(args.warmup, n_steps):
        e = ev[t]
        ph["refresh"] += e[0].elapsed_time(e[1]) / K
        ph["merge"] += e[1].elapsed_time(e[2]) / K
        for i in range(M):
            ph["sample"] += (e[2] if i == 0 else e[2 + 2 * i]).elapsed_time(e[3 + 2 * i]) / K
            ph["step"] += e[3 + 2 * i].elapsed_time(e[4 + 2 * i]) / K
    owned = [ids[(ids >= lo) & (ids < hi)] for ids in keep_ids]
    U = sum(int(torch.unique(o).numel()) for o in owned) / len(owned)
    slots = sum(int(o.numel()) for o in owned) / len(owned)
    gemm_ms, gemm_n = kt["refresh_gemm"]
    flops = 2.0 * Lr * d * Rg
    ach = flops / (gemm_ms / max(gemm_n, 1) / 1e3) / 1e12
    sgl_ms, sgl_n = kt["step_single"]
    upd_bytes = U * d * 8
    # what rank 0 would send/receive per step in the real job (bytes, per rank)
    coll = {
        "queries_all_gather": (N - 1) * R * d * 4,
        "positives_all_gather": (N - 1) * R * (lpp * 4 + 8),
        "keys_all_to_all": (N - 1) * R * k_h * 8,
        **({"bf16_candidate_keys_all_to_all": (N - 1) * R * kc * 8, "tau_all_gather": (N - 1) * R * 8}
           if global_rr else {}),
        **({"sample_stats_all_to_all": (N - 1) * R * j_sh * 4, "candidate_tau_all_gather": (N - 1) * R * 8,
            "candidate_counts_all_to_all": (N - 1) * R * 16, "verify_flags_all_gather": (N - 1) * R * 4}
           if j_sh > 0 else {}),
        **({"sampler_inputs_all_gather": M * (N - 1) * B * (8 + lpp * 4 + 8 + k_h * 4)} if regen else
           {"slates_all_gather": M * (N - 1) * B * S * 10}),
        "emb_all_gather": M * (N - 1) * B * d * 4,
        "grad_emb_reduce_scatter": M * (N - 1) * B * d * 4,
        "loss_status_all_reduce": M * 2 * (8 + 16),
    }
    line = {
        "metric": METRIC + f" [emulated {N}-GPU job: rank 0's compute on 1 GPU, collectives not run]",
        "value": round(Rg * K / (ms * K / 1e3), 1), "unit": UNIT, "n_gpus": 1, "emulates_n_gpus": N,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32 W/step, bf16 tensor-core refresh + fp32 re-rank", "data": "synthetic",
        "config": dict(bench_config(N), labels_shard=Lr, rows_per_step_job=Rg, minibatch_job=Bg,
                       slate_exchange=args.slate_exchange,
                       sharded_rerank=("global k'-th bf16 key threshold (engine._refresh_sharded_rerank; "
                                       "tau proxied by this shard's ceil(k'/N)-th key)") if global_rr
                       else "every shard re-ranks its full local top-k'",
                       sharded_candidates=("global threshold from the shards' sample statistics "
                                           "(engine._candidates_global; the global j-th sampled maximum proxied by "
                                           "this shard's ceil(j/N)-th, the verify set by count x N < k')")
                       if j_sh > 0 else "each shard's own top-k' candidates"),
        "phases_ms_per_step": {k: round(v, 4) for k, v in ph.items()},
        "owned_slots_per_minibatch": round(slots, 1), "unique_owned_labels_per_minibatch": round(U, 1),
        "occurrences_per_owned_label": round(slots / max(U, 1), 3),
        "roofline": {"bound": "tensor", "kernel": "refresh_tc_kernel threshold pass", "achieved": round(ach, 2),
                     "peak": tf_burst, "unit": "TFLOP/s", "frac": round(ach / tf_burst, 4),
                     "launch_ms": round(gemm_ms / max(gemm_n, 1), 4), "peak_kind": f"{peak_kind} burst bf16"},
        "roofline_step": {"bound": "hbm", "kernel": "step_single", "launch_ms": round(sgl_ms / max(sgl_n, 1), 4),
                          "achieved": round(upd_bytes / (sgl_ms / max(sgl_n, 1) / 1e3) / 1e9, 1) if sgl_n else None,
                          "peak": hbm, "unit": "GB/s", "algorithmic": f"U*d*8 = {upd_bytes:.3e} B (U={U:.0f})"},
        "collective_bytes_per_rank_per_step": coll,
        "collective_bytes_total_per_rank_per_step": int(sum(coll.values())),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ C5 shard emulation
C5 = dict(workload="120M-label synthetic, rank-0 shard of 8 (15M labels) emulated on one GPU", L_total=120_000_000,
          world=8, d=768, B_global=4096, k_p=16, k_h=200, k_i=128, n_cand=128, k_r=2000, labels_per_point=10,
          lr=1e-3, wd=0.0)


def run_c5shard(args):
    """BASELINE.json configs[4] as one of its 8 label shards: W (15M x 768 bf16)
    + Adam m, v (fp32) resident on this GPU. Each step:
      refresh  the global batch's 4096 queries against the shard (bf16 tcgen05
               two-pass + re-rank on the bf16 rows) for top-(k_h + n_c) =
               top-328, then the merge of the 8 shards' lists (astra_topk_merge;
               the other 7 shards' lists are this shard's list relabelled into
               their label ranges, so the merged cache owns 1/8 of its ids here,
               as in the real job) and astra_importance_split: the negative-
               mixture cache H (k_h=200) + importance candidates C (n_c=128)
               with q = sigmoid(stale score). This refresh
               builds the NEXT step's cache (stale by one step).
      sample   Philox slates over all 120M labels from the previous refresh's
               cache: k_p=16, k_h=200, k_i=128 importance draws (weight
               1/(k_i q)), k_r=2000 uniform -> S=2344.
      step     the fused loss/Adam update of the slots this shard owns (~1/8).
    n_c = 128 (not 200): the bf16-row re-rank holds k' <= 512 candidates, so
    k_h + n_c <= 341. The collectives of the 8-GPU job (query / embedding
    all-gathers, key all-to-all, grad_emb reduce-scatter: ~40 MB per step over
    NVLink) are not run; the line reports the shard's compute time."""
    import torch

    from paper_2409_20156_b200 import _lib, ops

    torch.cuda.set_device(0)
    c = C5
    N = c["world"]
    L = c["L_total"] // N
    d, B = c["d"], c["B_global"]
    k_h, n_c, k_i = c["k_h"], c["n_cand"], c["k_i"]
    kc = k_h + n_c
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
    shift = torch.arange(N, dtype=torch.int64, device="cuda").view(N, 1, 1) * L  # label-range offsets of the shards

    def cache_of(emb, ip, pid):
        keys, _, _ = ops.refresh_topk(emb, ip, pid, kc, "bf16_rerank", labels_bf16=snap)
        # keys = (ord(score) << 32) | (2^32 - 1 - id): relabelling id -> id + s*L subtracts s*L
        _, gids, gscores = ops.topk_merge((keys.unsqueeze(0) - shift).contiguous(), kc)
        return ops.importance_split(gids, gscores, k_h)

    n_steps = args.warmup + args.steps
    data = []
    for t in range(n_steps):
        rows = torch.arange(t * B, (t + 1) * B, dtype=torch.int64, device="cuda")
        pos = torch.randint(0, c["L_total"], (B, c["labels_per_point"]), device="cuda", generator=g).sort(1).values
        ip = torch.arange(0, B * c["labels_per_point"] + 1, c["labels_per_point"], dtype=torch.int64, device="cuda")
        pid = pos.to(torch.int32).reshape(-1).contiguous()
        emb = torch.randn((B, d), device="cuda", generator=g)
        data.append([rows, ip, pid, emb, None])
    data[0][4] = cache_of(data[0][3], data[0][1], data[0][2])  # the first step's stale cache
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = [[_ev() for _ in range(4)] for _ in range(n_steps)]

    def one(t):
        rows, ip, pid, emb, cache = data[t]
        e = ev[t]
        e[0].record(stream)
        nxt = cache_of(emb, ip, pid)  # the next step's cache (stale by one step)
        if t + 1 < n_steps:
            data[t + 1][4] = nxt
        e[1].record(stream)
        hard, cand, cand_q = cache
        sl = ops.sample_slates(0, 1, t, rows, ip, pid, hard, k_h, c["L_total"], c["k_p"], c["k_r"], cand=cand,
                               cand_q=cand_q, k_i=k_i)
        e[2].record(stream)
        res = ops.slate_step(emb, *sl, W, c["lr"], c["wd"], optimizer="adam", adam_m=m, adam_v=v, adam_step=t + 1,
                             label_offset=0, w_absmax=w_absmax)
        e[3].record(stream)
        data[t][4] = None
        return res, sl

    for t in range(args.warmup):
        one(t)
    torch.cuda.synchronize()
    for name in ("refresh_gemm", "refresh_verify", "step_single", "slot_forward", "label_update"):
        _lib.kernel_timing(name)
    _lib.kernel_timing_enable(True)
    clocks = ClockSampler(0)
    clocks.start()
    t0, t1 = _ev(), _ev()
    t0.record(stream)
    for t in range(args.warmup, n_steps):
        res, sl = one(t)
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
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
    n_imp_owned = int(((sl[2] == ops.ORIGIN_IMP) & (ids >= 0) & (ids < L)).sum())
    hbm, tf_burst, tf_sus, peak_kind = peaks()
    gemm_ms, gemm_n = kt["refresh_gemm"]
    flops = 2.0 * L * d * B
    achieved = flops / (gemm_ms / max(gemm_n, 1) / 1e3) / 1e12
    step_bytes = U * d * (2 * 2 + 2 * 8) + 2 * B * d * 4 + B * sl[0].shape[1] * 5
    upd_ms, upd_n = kt["label_update"]
    sgl_ms, sgl_n = kt["step_single"]
    upd_bytes = U * d * (2 * 2 + 2 * 8)
    line = {
        "metric": METRIC + " [C5 shard emulation]", "value": round(B / (ms / 1e3), 1), "unit": UNIT, "n_gpus": 1,
        "emulates_n_gpus": N, "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16 W + fp32 Adam state; bf16 tcgen05 refresh + re-rank on the bf16 rows", "data": "synthetic",
        "config": {"workload": c["workload"], "n_labels_total": c["L_total"], "labels_shard": L, "dim": d,
                   "global_batch": B, "k_p": c["k_p"], "k_h": k_h, "k_i": k_i, "n_cand": n_c, "k_r": c["k_r"],
                   "slate": int(sl[0].shape[1]), "tau_r": 1, "optimizer": "adam", "owned_slots": int(own.numel()),
                   "owned_importance_slots": n_imp_owned, "unique_rows": U,
                   "importance_cache": "refresh top-(k_h+n_c) -> merge -> H + C, q = sigmoid(stale score)"},
        "phases_ms_per_step": {k: round(v, 3) for k, v in ph.items()},
        "refresh_mips_qps_shard": round(B / (ph["refresh"] / 1e3), 1),
        "refresh_verify_ms": round(kt["refresh_verify"][0] / max(kt["refresh_verify"][1], 1), 4),
        "composite_tau_r5_samples_per_s": round(B / ((ph["sample"] + ph["step"] + ph["refresh"] / 5) / 1e3), 1),
        "roofline": {"bound": "tensor", "kernel": "refresh_tc_kernel threshold pass", "achieved": round(achieved, 2),
                     "peak": tf_burst, "unit": "TFLOP/s", "frac": round(achieved / tf_burst, 4),
                     "frac_of_sustained_peak": round(achieved / tf_sus, 4),
                     "launch_ms": round(gemm_ms / max(gemm_n, 1), 3)},
        "roofline_step": {"bound": "hbm", "achieved": round(step_bytes / (ph["step"] / 1e3) / 1e9, 1), "peak": hbm,
                          "unit": "GB/s", "frac": round(step_bytes / (ph["step"] / 1e3) / 1e9 / hbm, 4),
                          "algorithmic": f"U*d*(2*2 + 2*8) + 2*B*d*4 + B*S*5 = {step_bytes:.3e} B (U={U})",
                          "label_update_launch_ms": round(upd_ms / max(upd_n, 1), 4) if upd_n and not sgl_n else None,
                          "kernels": {name: {"launch_ms": round(ms_ / n_, 4),
                                             "achieved_gbs": round(upd_bytes / (ms_ / n_ / 1e3) / 1e9, 1),
                                             "algorithmic_bytes": int(upd_bytes)}
                                      for name, (ms_, n_) in ((("step_single", (sgl_ms, sgl_n)),) if sgl_n else
                                                              (("label_update", (upd_ms, upd_n)),)) if n_}},
        "memory_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
        "clocks": clk,
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
    dense SGD of every row (G^T E) — three fp32-accurate GEMMs on the tf32
    tensor cores (astra_gemm_f32, 3xTF32) + astra_dense_bce / astra_dense_sgd —
    next to the oracle port of the same
    NumPy arithmetic on the host cores (one minibatch). The dense comparison
    for the sampled arm."""
    import torch

    from oracle import xcmix_port as port
    from paper_2409_20156_b200 import _lib, ops

    torch.cuda.set_device(0)
    hbm, tf_burst, tf_sus, peak_kind = peaks()
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
    _lib.kernel_timing("gemm_f32")
    _lib.kernel_timing_enable(True)
    a, b = _ev(), _ev()
    a.record(stream)
    for t in range(args.steps):
        loss = one(t)
    b.record(stream)
    torch.cuda.synchronize()
    _lib.kernel_timing_enable(False)
    gemm_ms, gemm_n = _lib.kernel_timing("gemm_f32")
    ms = a.elapsed_time(b) / args.steps
    flops = 3 * 2.0 * B * L * d
    # the GEMM kernel issues 3 tf32 products per fp32 product (hi*hi + lo*hi + hi*lo):
    # tensor work = 3 x the algorithmic flops; the tf32 dense rate is half the bf16 one
    t_gemm = gemm_ms / max(gemm_n, 1) / 1e3
    tf32_peak = tf_burst / 2
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
        "dtype": "fp32-accurate GEMMs on the tf32 tensor cores (3xTF32 split, astra_gemm_f32) + float64 loss",
        "data": "synthetic",
        "config": {"workload": "train_full_loss_baseline at the reference's label cap", "n_labels": L, "dim": d,
                   "minibatch": B, "labels_per_point": lpp},
        "fp32_equivalent_tflops": round(flops / (ms / 1e3) / 1e12, 2),
        "roofline": {"bound": "tensor", "kernel": "gemm_f32 (tcgen05 kind::tf32, CTA pairs, 3 products per fp32 product)",
                     "achieved": round(flops / t_gemm / 1e12, 2) if gemm_n else None,
                     "peak": round(tf32_peak, 1), "unit": "TFLOP/s",
                     "frac": round(flops / t_gemm / 1e12 / tf32_peak, 4) if gemm_n else None,
                     "traffic": None,
                     "algorithmic": f"3 GEMMs x 2*B*L*d = {flops:.3e} fp32 flop per step = 3x that in tf32 MMA work; "
                                    "achieved = tf32 MMA flops of one launch (3 x 2*M*N*K) / its duration",
                     "launch_ms": round(t_gemm * 1e3, 4) if gemm_n else None,
                     "peak_kind": f"{peak_kind} burst bf16 / 2 (tf32 dense rate)"},
        "cpu_baseline": {"value": round(B / t_cpu, 2), "unit": "samples/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": "one minibatch of the NumPy arm (oracle port), threads=all"},
    }
    print(json.dumps(line), flush=True)


def run_dropin(args):
    """The C4 work through the REFERENCE's own public API with the B200 path
    installed (paper_2409_20156_b200.install: xcmix.anns.retrieve_hard_negatives
    and xcmix.trainer._batch_forward_backward rebound), on the same state the
    reference arm builds (ReferenceCPU: TrainerState, the reference's encoder
    on the host). Per step: the refresh of one B=1024 minibatch's rows through
    xcmix.anns.retrieve_hard_negatives (host numpy in, NegativeCache out) + the
    minibatch's xcmix.trainer._batch_forward_backward (slates, fused loss /
    update on the device-resident W, grad_emb back to the caller's numpy
    encoder + Adam) — exactly the reference arm's step, so the two lines compare
    the same calls. Host-synchronous API: timed by wall clock with the device
    synchronised on both sides (the numbers include every H2D / D2H)."""
    import torch

    from paper_2409_20156_b200 import _lib
    from paper_2409_20156_b200.install import install

    torch.cuda.set_device(0)
    B = CFG["B"]
    n_steps = args.warmup + args.steps
    ref = ReferenceCPU(B * n_steps)
    if ref.kind != "reference":
        print(json.dumps({"metric": METRIC + " [through the reference API]", "unavailable": "baseline/_ref missing"}))
        return
    install(slates="philox")
    from xcmix import anns
    from xcmix import trainer as xt

    ref.index = anns.build_exact(ref.state.bank.weights, snapshot_epoch=0)  # the rebound (device-cached) snapshot
    # the caller's host encoder (numpy forward / backward / Adam, outside the
    # hot path) is timed separately so the line shows what the drop-in's own
    # calls cost
    enc_s = [0.0]

    def timed(fn):
        def w(*a, **k):
            t = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                enc_s[0] += time.perf_counter() - t
        return w

    for name in ("embed_batch", "encoder_backward_batch", "adam_step"):
        setattr(xt, name, timed(getattr(xt, name)))

    def step(t):
        rows = t * B + np.arange(B, dtype=np.int64)
        pos = [ref.positives[r] for r in rows]
        emb = xt.embed_batch(ref.state.encoder, ref.state.dataset.features[rows])
        cache = anns.retrieve_hard_negatives(ref.index, emb, pos, CFG["k_h"])
        ref.cache_ids[rows] = cache.ids
        return xt._batch_forward_backward(ref.state, rows, 2, np.random.default_rng(1000 + t), 0.01, CFG["lr"])

    for t in range(args.warmup):
        step(t)
    torch.cuda.synchronize()
    n0 = _lib.launch_count()
    enc_s[0] = 0.0
    prof = None
    if os.environ.get("ASTRA_BENCH_PROFILE"):  # host profile of the timed steps (diagnosis)
        import cProfile

        prof = cProfile.Profile()
        prof.enable()
    t0 = time.perf_counter()
    for t in range(args.warmup, n_steps):
        loss = step(t)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if prof is not None:
        import pstats

        prof.disable()
        pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(25)
    K = args.steps
    line = {"metric": METRIC + " [through the reference API: install() + xcmix functions]",
            "value": round(B * K / wall, 1), "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": args.warmup,
            "ms_per_step": round(wall / K * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp32 W/step, bf16 tensor-core refresh + fp32 re-rank; deterministic two-kernel step",
            "data": "synthetic",
            "config": dict(bench_config(1), rows_per_step_per_gpu=B, minibatches_per_step=1, refresh_chunk=B,
                           api="xcmix.anns.retrieve_hard_negatives + xcmix.trainer._batch_forward_backward"),
            "timing": "wall clock, device synchronised on both sides (host-synchronous API, numpy in/out)",
            "host_encoder_ms_per_step": round(enc_s[0] / K * 1e3, 3),
            "classifier_path_ms_per_step": round((wall - enc_s[0]) / K * 1e3, 3),
            "note": "host_encoder = the caller's numpy encoder (xcmix.trainer.embed_batch / encoder_backward_batch / "
                    "adam_step on the host cores, outside the hot path); classifier_path = everything else: the "
                    "refresh, slates, fused step and their host<->device copies",
            "gpu_launches": int(_lib.launch_count() - n0), "last_loss": float(loss)}
    print(json.dumps(line), flush=True)


def _relaunch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-exec under
    torch.distributed.run with one rank per GPU (NCCL), same arguments."""
    import torch

    have = torch.cuda.device_count()
    if have < n:
        sys.exit(f"bench.py: --gpus {n} requested but only {have} CUDA device(s) are visible")
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "WARN"))
    sys.stderr.write(f"[bench] launching {n} ranks: {' '.join(cmd)}\n")
    rc = subprocess.call(cmd, env=env)
    if rc:
        sys.exit(rc)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c4", choices=["c4", "c1", "c2", "c3", "c5shard", "fullloss", "dropin"],
                    help="c4 (default, the headline line); c1 / c2 / c3 (BASELINE configs[0..2], same composite "
                         "step); c5shard (120M-label config, one of 8 shards); fullloss (the all-negatives arm at the "
                         "reference's 50K-label cap); dropin (the same C4 work through the reference's own API with "
                         "install())")
    ap.add_argument("--refresh-sms", type=int, default=0,
                    help="SM budget of the refresh running concurrently with training on a side stream (0 = serial)")
    ap.add_argument("--emulate-shard-candidates", action="store_true",
                    help="--emulate: each shard finds its own top-k' candidates (no global candidate threshold)")
    ap.add_argument("--emulate-full-rerank", action="store_true",
                    help="--emulate: every shard re-ranks its full local top-k' (no global threshold)")
    ap.add_argument("--emulate", type=int, default=0,
                    help="one GPU runs rank 0's share of an N-GPU C4 job (a 1/N label shard, all N ranks' rows); "
                         "collectives are not run, their bytes are reported")
    ap.add_argument("--w-init", default="uniform", choices=["uniform", "clustered"],
                    help="C4 line: W uniform-scaled (the reference's init) or trained-like clustered heavy-tailed "
                         "with duplicated rows and queries near popular clusters (exercises the refresh's "
                         "overflow -> exact verify path)")
    ap.add_argument("--refresh-mode", default="bf16_rerank", choices=["bf16_rerank", "fp8_rerank"],
                    help="tensor-core candidate pass of the refresh (bf16 = the north star's, or e4m3 at twice the "
                         "tensor rate), then the fp32-exact re-rank")
    ap.add_argument("--no-alt-fp8", action="store_true", help="skip the e4m3-refresh comparison object")
    ap.add_argument("--slate-exchange", default="gather", choices=["gather", "regenerate"],
                    help="--emulate: how the N-GPU job shares slates (engine.ClassifierEngine.slate_exchange)")
    args = ap.parse_args()
    # no cyclic-GC pauses inside the timed regions (a generation-2 collection
    # takes 18-37 ms in this process); reference counting still frees memory
    gc.collect()
    if os.environ.get("ASTRA_BENCH_GC"):  # diagnosis: keep GC on, log every collection's duration
        _gc_t = {}

        def _gc_log(phase, info):
            if phase == "start":
                _gc_t["t"] = time.perf_counter()
            else:
                print(f"gc gen{info['generation']} {1e3 * (time.perf_counter() - _gc_t['t']):.2f} ms", file=sys.stderr)

        gc.callbacks.append(_gc_log)
    else:
        gc.disable()
    REFRESH_MODE[0] = args.refresh_mode
    if args.config in CONFIGS:
        CFG.clear()
        CFG.update(CONFIGS[args.config])
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    env_world = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and env_world is None and args.impl == "ours":
        # launched without torchrun: start one rank per GPU ourselves
        return _relaunch(args.gpus)
    if env_world is not None and int(env_world) != args.gpus and args.impl == "ours":
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}; refusing to report a different GPU count")
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "dropin":
        run_dropin(args)
    elif args.emulate:
        run_emulate(args)
    elif args.config == "c5shard":
        run_c5shard(args)
    elif args.config == "fullloss":
        run_fullloss(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
