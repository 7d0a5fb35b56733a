"""Device-resident ASTRA classifier state and the full classifier step.

`ClassifierEngine` owns one label shard of W (+ optimizer state) on one GPU
and runs the hot path of SURVEY.md §8:

  snapshot()  build_exact (anns.py:99): an immutable fp32 copy of W plus its
              bf16 copy for the tensor-core refresh; non-finite -> NumericalError.
  refresh()   retrieve_hard_negatives (anns.py:233-256) over every shard:
              local fused GEMM + top-k, all-gather of partial keys, exact merge.
  sample()    _assemble_batch_slates (trainer.py:262-318) via Philox.
  step()      classifier half of _batch_forward_backward (trainer.py:366-394):
              fused loss fwd/bwd + sparse SGD/Adam update of the local shard,
              grad_emb reduce-scattered back to the rows' owners.
  train_step_host()  the end-to-end call with HOST buffers (pinned H2D of the
              step's inputs, D2H of grad_emb / loss / refreshed ids).

All device work goes through `backend` (default: the CUDA C-ABI ops module).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import ops as cuda_ops
from .errors import ConfigError, DataError, NumericalError
from .shard import Comm, gather_csr, shard_range


def init_uniform_scaled(rows: int, dim: int, seed: int, device) -> torch.Tensor:
    """uniform(-1/sqrt(d), 1/sqrt(d)) like init_classifiers (classifiers.py:37-40),
    drawn on the device (torch generator, not NumPy's PCG64 stream)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    bound = 1.0 / math.sqrt(dim)
    w = torch.empty((rows, dim), dtype=torch.float32, device=device)
    w.uniform_(-bound, bound, generator=g)
    return w


class ClassifierEngine:
    def __init__(self, n_labels: int, dim: int, *, k_p: int, k_h: int, k_r: int, k_i: int = 0, n_c: int = 0,
                 weights=None, w_dtype=torch.float32, optimizer: str = "sgd", betas=(0.9, 0.999), eps=1e-8,
                 refresh_mode: str = "bf16_rerank", seed: int = 0, device=None, group=None, backend=None):
        if optimizer not in ("sgd", "adam"):
            raise ConfigError(f"unknown optimizer {optimizer!r}")
        if k_p < 1 or k_h < 0 or k_r < 0 or k_i < 0 or n_c < 0:
            raise ConfigError("need k_p >= 1, k_h >= 0, k_r >= 0, k_i >= 0, n_c >= 0")
        if k_i > 0 and n_c == 0:
            raise ConfigError("importance draws (k_i > 0) need n_c > 0 candidates per row")
        self.ops = backend if backend is not None else cuda_ops
        self.comm = Comm(group)
        self.device = torch.device(device if device is not None else ("cuda" if torch.cuda.is_available() else "cpu"))
        self.n_labels, self.dim = int(n_labels), int(dim)
        self.lo, self.hi = shard_range(self.n_labels, self.comm.rank, self.comm.world)
        self.k_p, self.k_h, self.k_r, self.k_i, self.n_c = k_p, k_h, k_r, k_i, n_c
        self.seed = seed
        self.refresh_mode = refresh_mode
        self.optimizer = optimizer
        self.betas, self.eps = betas, eps
        if weights is None:
            W = init_uniform_scaled(self.hi - self.lo, dim, seed + 1 + 7919 * self.comm.rank, self.device)
        else:
            W = torch.as_tensor(weights)[self.lo : self.hi].to(self.device, torch.float32)
        self.W = W.to(w_dtype).contiguous()
        # running bound on max|W| (kept current by every update): lets the step
        # prove finiteness up front and take the single label-major step pass
        self.w_absmax = self.W.abs().amax().float().reshape(1).clone() if self.W.numel() else \
            torch.zeros(1, dtype=torch.float32, device=self.device)
        self.m = self.v = None
        if optimizer == "adam":
            self.m = torch.zeros((self.hi - self.lo, dim), dtype=torch.float32, device=self.device)
            self.v = torch.zeros_like(self.m)
        self.adam_step = 0
        self.snap_f32 = self.snap_bf16 = self.snap_f8 = None
        self.snapshot_epoch = -1
        self.slate_exchange = "gather"  # or "regenerate" (see sample())
        # BF16_RERANK over shards: re-rank only the candidates at or above the
        # global k'-th bf16 key (_refresh_sharded_rerank); False: every shard
        # re-ranks its full local top-k'
        self.global_rerank_threshold = True
        # ... and its bf16 candidate pass with a global threshold from the
        # shards' sample statistics (_candidates_global); False: each shard
        # finds its own top-k' candidates
        self.global_candidate_threshold = True
        self._shard_plan = {}
        # cross-rank reduction of grad_emb and the loss in step(): "collective"
        # = reduce_scatter / all_reduce (NCCL's order); "ordered" = every
        # rank's partials sent to the rows' owners (all_to_all) and summed in
        # rank order 0..G-1, so with astra_set_step_deterministic(1) a sharded
        # run is bitwise reproducible (SURVEY §8e's fixed-order option)
        self.grad_reduce = "collective"
        # W writes since construction; an aliased snapshot (snapshot(copy=False))
        # is valid only while this matches the value it was taken at
        self._w_version = 0
        self._snap_alias_version = None

    # ------------------------------------------------------------ snapshot
    def snapshot(self, epoch: int = 0, check_finite: bool = True, copy: bool = True) -> None:
        """Immutable copy of the shard for the refresh (anns.py:90-100).

        copy=False is the synchronous-refresh form: the snapshot
        aliases the live W instead of copying it (no 4 GB fp32 copy at C4, no
        23 GB bf16 copy on a C5 shard; the tensor-core copy is still built when
        W is fp32), for a caller that runs every refresh of this snapshot
        before the next update. refresh() raises ConfigError once W has been
        written after an aliased snapshot."""
        if check_finite and not bool(torch.isfinite(self.W).all()):
            raise NumericalError("non-finite vectors in index build")
        fp8 = self.refresh_mode == "fp8_rerank"
        self._snap_alias_version = None if copy else self._w_version
        if self.W.dtype == torch.bfloat16 and self.refresh_mode != "fp32":
            # bf16 W: the bf16 copy is the whole snapshot (the re-rank scores its
            # values exactly); no fp32 copy (46 GB for a 15M-label shard)
            self.snap_f32 = None
            self.snap_bf16 = self.W.clone() if copy else self.W
        else:
            if self.W.dtype != torch.float32:
                self.snap_f32 = self.W.float()
            else:
                self.snap_f32 = self.W.clone() if copy else self.W
            self.snap_bf16 = (self.ops.f32_to_bf16(self.snap_f32) if self.refresh_mode in ("bf16", "bf16_rerank")
                              else None)
        # e4m3 candidate-pass snapshot (FP8_RERANK: the re-rank reads the fp32 / bf16 copy above)
        self.snap_f8 = (self.ops.quantize_e4m3(self.snap_f32 if self.snap_f32 is not None else self.snap_bf16)
                        if fp8 else None)
        self.snapshot_epoch = epoch

    # ------------------------------------------------------------ refresh
    def refresh(self, queries: torch.Tensor, pos_indptr: torch.Tensor, pos_ids: torch.Tensor, k: int,
                mode: str | None = None):
        """Global top-k (ids, scores) for this rank's queries over ALL shards,
        positives excluded. Collective when world_size > 1."""
        if self.snap_f32 is None and self.snap_bf16 is None:
            raise ConfigError("refresh before snapshot()")
        if self._snap_alias_version is not None and self._snap_alias_version != self._w_version:
            raise ConfigError("W was updated after an aliased snapshot(copy=False); take a new snapshot")
        mode = mode or self.refresh_mode
        B = queries.shape[0]
        q_all = self.comm.all_gather(queries)
        ip_all, pid_all = gather_csr(self.comm, pos_indptr, pos_ids)
        if self.comm.world > 1 and mode == "bf16_rerank" and self.global_rerank_threshold and self.snap_bf16 is not None:
            return self._refresh_sharded_rerank(q_all, ip_all, pid_all, k)
        extra = {"labels_e4m3": self.snap_f8} if getattr(self, "snap_f8", None) is not None else {}
        keys, ids, scores = self.ops.refresh_topk(
            q_all, ip_all, pid_all, k, mode, labels_f32=self.snap_f32, labels_bf16=self.snap_bf16, label_offset=self.lo,
            **extra)
        if self.comm.world == 1:
            return ids, scores
        # rows [r*B, (r+1)*B) of every shard's partial list go to their owner r
        mine = self.comm.all_to_all(keys)  # [world, B, k]: shard i's keys for this rank's rows
        _, ids, scores = self.ops.topk_merge(mine, k)
        return ids, scores

    def _refresh_sharded_rerank(self, q_all, ip_all, pid_all, k):
        """BF16_RERANK over label shards with a global candidate threshold.
        Each shard's bf16 top-k' (k' = rerank_candidates_count(k)) goes to the
        rows' owners, which merge the world lists and return the global k'-th
        bf16 key tau per row; each shard then re-ranks in fp32 only its
        candidates with key >= tau (~k'/world per row instead of k'), and the
        fp32 partial top-k lists are merged as before. The re-ranked set is the
        global bf16 top-k' — the single-GPU candidate set — so the result is
        the single-GPU BF16_RERANK result, with the fp32 re-rank work no longer
        growing with the world size."""
        kc = self.ops.rerank_candidates_count(k)
        j = self._sharded_plan_j(q_all.shape[0], kc) if self.global_candidate_threshold else 0
        if j > 0:
            ckeys = self._candidates_global(q_all, ip_all, pid_all, kc, j)
        else:
            ckeys, _, _ = self.ops.refresh_topk(q_all, ip_all, pid_all, kc, "bf16", labels_f32=self.snap_f32,
                                                labels_bf16=self.snap_bf16, label_offset=self.lo)
        merged, _, _ = self.ops.topk_merge(self.comm.all_to_all(ckeys), kc)  # [B, kc]: this rank's rows
        tau_all = self.comm.all_gather(merged[:, kc - 1].contiguous())     # [world*B]; 0: fewer than k' exist
        flip = torch.tensor(-(2 ** 63), dtype=torch.int64, device=ckeys.device)  # unsigned order of the keys
        keep = (ckeys ^ flip) >= (tau_all[:, None] ^ flip)
        cand = torch.where(keep, ckeys, torch.zeros_like(ckeys))
        fkeys, _, _ = self.ops.rerank_candidates(q_all, cand, k, labels_f32=self.snap_f32,
                                                 labels_bf16=self.snap_bf16 if self.snap_f32 is None else None,
                                                 label_offset=self.lo)
        _, ids, scores = self.ops.topk_merge(self.comm.all_to_all(fkeys), k)
        return ids, scores

    def _sharded_plan_j(self, nq_all: int, kc: int) -> int:
        """j of the sharded candidate pass's sample statistics, agreed by every
        rank (0: some shard's shape does not run the two-pass plan, so all take
        the per-shard candidate pass). One collective per shape, cached."""
        key = (nq_all, kc)
        if key not in self._shard_plan:
            j = int(self.ops.refresh_plan_j(nq_all, self.hi - self.lo, self.dim, kc))
            t = torch.tensor([j, -j], dtype=torch.int64, device=self.device)
            self.comm.all_reduce(t, op="min")
            jmin, jmax = int(t[0]), -int(t[1])
            self._shard_plan[key] = jmin if jmin == jmax and jmin > 0 else 0
        return self._shard_plan[key]

    def _candidates_global(self, q_all, ip_all, pid_all, kc, j):
        """The shard's bf16 candidates (top-k' of its labels that can be in the
        global top-k', positives excluded) with a GLOBAL threshold: the rows'
        owners take the j-th largest sampled group maximum over all shards'
        sample statistics (so the threshold pass appends ~k'/world candidates
        per query per shard instead of ~k'), sum the shards' candidate counts
        and send back which queries lack k' candidates globally (or overflowed
        a list); those run the exact verify pass on every shard. The union of
        the shards' lists contains the global top-k' for every query."""
        ops, comm = self.ops, self.comm
        B = q_all.shape[0] // comm.world
        top = ops.refresh_sharded_stage(1, q_all, ip_all, pid_all, kc, self.snap_bf16, label_offset=self.lo)
        mine = comm.all_to_all(top.to(torch.int64) & 0xFFFFFFFF)            # [world, B, j]
        gj = mine.permute(1, 0, 2).reshape(B, -1).topk(j, dim=1).values[:, j - 1]
        tau_all = comm.all_gather(gj << 32)                                  # [world*B] key form
        keys, counts, oflow = ops.refresh_sharded_stage(2, q_all, ip_all, pid_all, kc, self.snap_bf16,
                                                        label_offset=self.lo, tau_keys=tau_all)
        cnt = comm.all_to_all(counts.to(torch.int64)).sum(0)                 # [B]
        ovf = comm.all_to_all(oflow.to(torch.int64)).amax(0)
        need = comm.all_gather(((cnt < kc) | (ovf > 0)).to(torch.int32))    # [world*B]
        return ops.refresh_sharded_stage(3, q_all, ip_all, pid_all, kc, self.snap_bf16, label_offset=self.lo,
                                         io_keys=keys, flags=need)

    def refresh_cache(self, queries: torch.Tensor, pos_indptr: torch.Tensor, pos_ids: torch.Tensor,
                      mode: str | None = None):
        """The negative-mixture cache rows of this rank's queries from one
        stale refresh: (hard [B, k_h], cand [B, n_c],
        cand_q [B, n_c]) — H = the top k_h, the importance candidates C = the
        next n_c with stored draw weights sigmoid(stale score)
        (astra_importance_split). Without the importance class (k_i == 0)
        cand / cand_q are None and this is refresh(k_h)."""
        if self.k_i == 0:
            ids, _ = self.refresh(queries, pos_indptr, pos_ids, self.k_h, mode)
            return ids, None, None
        ids, scores = self.refresh(queries, pos_indptr, pos_ids, self.k_h + self.n_c, mode)
        return self.ops.importance_split(ids, scores, self.k_h)

    # ------------------------------------------------------------ sampler
    def sample(self, rows, pos_indptr, pos_ids, hard, epoch: int, step: int, k_h: int | None = None,
               k_r: int | None = None, cand=None, cand_q=None):
        """Slates of the rows of ALL ranks (Philox, keyed by global row id,
        so every rank holds the same global slates as a 1-GPU run).
        slate_exchange (attribute):
          "gather" (default): each rank samples its own rows and the B x S
            slates are all-gathered (10 B per slot: 6 MB per rank at C4);
          "regenerate": the sampler's inputs (rows, positives, hard-cache
            rows, candidates; ~0.4 MB per rank at C4) are all-gathered and
            every rank draws all N x B rows itself.
        Measured (bench.py --emulate N, profiles/r02): regenerating costs
        0.39 / 0.62 / 1.04 ms per minibatch at N = 2 / 4 / 8 against 0.24 ms
        for the rank's own rows, more than the all-gather of the slates over
        NVLink (42 MB at N = 8), so "gather" is the default."""
        k_h = self.k_h if k_h is None else k_h
        k_r = self.k_r if k_r is None else k_r
        k_i = self.k_i if cand is not None else 0
        if self.comm.world > 1 and self.slate_exchange == "regenerate":
            rows = self.comm.all_gather(rows)
            pos_indptr, pos_ids = gather_csr(self.comm, pos_indptr, pos_ids)
            hard = self.comm.all_gather(hard) if hard is not None else None
            if cand is not None:
                cand, cand_q = self.comm.all_gather(cand), self.comm.all_gather(cand_q)
            return self.ops.sample_slates(self.seed, epoch, step, rows, pos_indptr, pos_ids, hard, k_h, self.n_labels,
                                          self.k_p, k_r, cand=cand, cand_q=cand_q, k_i=k_i)
        ids, y, origin, weights = self.ops.sample_slates(
            self.seed, epoch, step, rows, pos_indptr, pos_ids, hard, k_h, self.n_labels, self.k_p, k_r,
            cand=cand, cand_q=cand_q, k_i=k_i)
        if self.comm.world > 1:
            ids, y, origin, weights = (self.comm.all_gather(t) for t in (ids, y, origin, weights))
        return ids, y, origin, weights

    # ------------------------------------------------------------ step
    def step(self, emb: torch.Tensor, slates, lr: float, weight_decay: float, keep=None, factors_in=None):
        """Fused sampled-BCE step on this shard. Returns (loss_dev fp64[1],
        grad_emb of this rank's rows, status int32[4]). No host sync.
        Finiteness (classifiers.py:79-80: nothing written on a non-finite
        gradient) is guaranteed per shard: each shard checks its own rows'
        gradients before writing them; the all-reduced status reports a
        failure on any shard, but another shard may have applied its (finite)
        rows by then."""
        ids, y, origin, weights = slates
        emb_all = self.comm.all_gather(emb)
        keep_all = self.comm.all_gather(keep) if keep is not None else None
        if self.optimizer == "adam":
            self.adam_step += 1
        self._w_version += 1
        res = self.ops.slate_step(
            emb_all, ids, y, origin, weights, self.W, lr, weight_decay, keep=keep_all, factors_in=factors_in,
            optimizer=self.optimizer, adam_m=self.m, adam_v=self.v, adam_step=max(self.adam_step, 1),
            betas=self.betas, eps=self.eps, label_offset=self.lo, w_absmax=self.w_absmax)
        if self.grad_reduce == "ordered" and self.comm.world > 1:
            grad_emb = _sum_in_rank_order(self.comm.all_to_all(res.grad_emb))
            loss = _sum_in_rank_order(self.comm.all_gather_stack(res.loss_dev))
        else:
            grad_emb = self.comm.reduce_scatter(res.grad_emb)
            loss = self.comm.all_reduce(res.loss_dev)
        status = self.comm.all_reduce(res.status)
        return loss, grad_emb, status

    # ------------------------------------------------------------ host API
    def refresh_host(self, queries_h, pos_indptr_h, pos_ids_h, k: int | None = None, out=None):
        """retrieve_hard_negatives for a chunk of queries given in HOST (pinned)
        memory: H2D of the queries and positives, refresh, D2H of the ids.
        On CUDA the copies run on side streams (double-buffered staging), so
        they overlap the previous call's compute; `wait_host_outputs()` makes
        the current stream wait for the D2H."""
        if self.device.type != "cuda":
            ids, _ = self.refresh(queries_h.to(self.device), pos_indptr_h.to(self.device), pos_ids_h.to(self.device),
                                  k or self.k_h)
            out = torch.empty(ids.shape, dtype=ids.dtype) if out is None else out
            out.copy_(ids)
            return out
        pipe = self._pipe("refresh")
        d, slot = pipe.stage({"q": queries_h, "ip": pos_indptr_h, "pid": pos_ids_h})
        ids, _ = self.refresh(d["q"], d["ip"], d["pid"], k or self.k_h)
        pipe.release(slot)
        if out is None:
            out = torch.empty(ids.shape, dtype=ids.dtype, pin_memory=True)
        pipe.fetch(ids, out)
        return out

    def train_step_host(self, emb_h, rows_h, pos_indptr_h, pos_ids_h, hard_h, epoch, step, lr, weight_decay,
                        out=None, cand_h=None, cand_q_h=None):
        """One training minibatch with HOST inputs: H2D (pinned) of embeddings /
        rows / positives / hard-cache rows, Philox slates, fused loss + update,
        D2H of grad_emb and the loss. On CUDA the H2D copies of call i+1 run on
        a copy stream while call i computes (double-buffered device staging)
        and the D2H on a third stream; `wait_host_outputs()` orders them
        before the caller reads `out`. Returns ((grad_emb_h, loss_h), status_dev)."""
        if self.device.type != "cuda":
            dev = self.device
            hard = hard_h.to(dev) if hard_h is not None else None
            cand = cand_h.to(dev) if cand_h is not None else None
            cand_q = cand_q_h.to(dev) if cand_q_h is not None else None
            slates = self.sample(rows_h.to(dev), pos_indptr_h.to(dev), pos_ids_h.to(dev), hard, epoch, step,
                                 cand=cand, cand_q=cand_q)
            loss, grad_emb, status = self.step(emb_h.to(dev), slates, lr, weight_decay)
            if out is None:
                out = (torch.empty(grad_emb.shape, dtype=grad_emb.dtype), torch.empty(1, dtype=torch.float64))
            out[0].copy_(grad_emb)
            out[1].copy_(loss)
            return out, status
        pipe = self._pipe("step")
        d, slot = pipe.stage({"emb": emb_h, "rows": rows_h, "ip": pos_indptr_h, "pid": pos_ids_h, "hard": hard_h,
                              "cand": cand_h, "cand_q": cand_q_h})
        slates = self.sample(d["rows"], d["ip"], d["pid"], d["hard"], epoch, step, cand=d["cand"], cand_q=d["cand_q"])
        loss, grad_emb, status = self.step(d["emb"], slates, lr, weight_decay)
        pipe.release(slot)
        if out is None:
            out = (torch.empty(grad_emb.shape, dtype=grad_emb.dtype, pin_memory=True),
                   torch.empty(1, dtype=torch.float64, pin_memory=True))
        pipe.fetch(grad_emb, out[0])
        pipe.fetch(loss, out[1])
        return out, status

    def wait_host_outputs(self) -> None:
        """Make the current stream wait for every D2H issued by the host API.
        This only orders the streams: the host may read the `out` buffers
        after a synchronize of the current stream (or of an event recorded on
        it after this call)."""
        for pipe in getattr(self, "_pipes", {}).values():
            torch.cuda.current_stream().wait_stream(pipe.d2h)

    def _pipe(self, name: str) -> "_HostPipe":
        pipes = self.__dict__.setdefault("_pipes", {})
        if name not in pipes:
            pipes[name] = _HostPipe(self.device)
        return pipes[name]

    # ------------------------------------------------------------ host views
    def weights_host(self) -> np.ndarray:
        """This shard's W as fp32 NumPy (for eval / checkpoint boundaries)."""
        return self.W.float().cpu().numpy()

    # ------------------------------------------------------------ checkpoint
    _CKPT_MAGIC = b"XASH"
    _CKPT_VERSION = 1
    _CKPT_HEAD = "<4sIIIqqqiiiqfq"

    def save_shard(self, path: str) -> str:
        """Write this rank's shard — W in its own dtype, the Adam moments and
        step, the running max|W| bound — to `path` (+ ".rank{r}" when
        world > 1): the GPU-resident state the reference never checkpoints
        (its XAST file, trainer.py:689-710, holds the fp32 weights only; the
        full fp32 W for it is `weights_host()` gathered over the ranks).
        Little-endian header: magic, version, rank, world, n_labels, lo, hi,
        dim, w_dtype (0 fp32 / 1 bf16), optimizer (0 sgd / 1 adam),
        adam_step, w_absmax, snapshot_epoch; then W, m, v row-major."""
        import struct

        fn = path if self.comm.world == 1 else f"{path}.rank{self.comm.rank}"
        bf16 = self.W.dtype == torch.bfloat16
        adam = self.optimizer == "adam"
        head = struct.pack(self._CKPT_HEAD, self._CKPT_MAGIC, self._CKPT_VERSION, self.comm.rank, self.comm.world,
                           self.n_labels, self.lo, self.hi, self.dim, int(bf16), int(adam), self.adam_step,
                           float(self.w_absmax.item()), self.snapshot_epoch)
        with open(fn, "wb") as fh:
            fh.write(head)
            w = self.W.contiguous().view(torch.int16) if bf16 else self.W.contiguous()
            fh.write(w.cpu().numpy().tobytes())
            if adam:
                fh.write(self.m.cpu().numpy().tobytes())
                fh.write(self.v.cpu().numpy().tobytes())
        return fn

    def load_shard(self, path: str) -> None:
        """Restore a `save_shard` file into this engine (same shape, dtype,
        optimizer and rank layout); raises ConfigError/DataError on mismatch."""
        import struct

        fn = path if self.comm.world == 1 else f"{path}.rank{self.comm.rank}"
        hsize = struct.calcsize(self._CKPT_HEAD)
        import os

        fsize = os.path.getsize(fn)
        with open(fn, "rb") as fh:
            head = fh.read(hsize)
            if len(head) != hsize:
                raise DataError("truncated shard checkpoint")
            (magic, version, rank, world, n_labels, lo, hi, dim, bf16, adam, adam_step, w_absmax,
             snap) = struct.unpack(self._CKPT_HEAD, head)
            if magic != self._CKPT_MAGIC:
                raise DataError("bad shard checkpoint magic")
            if version != self._CKPT_VERSION:
                raise DataError(f"unsupported shard checkpoint version {version}")
            if (rank, world, n_labels, lo, hi, dim) != (self.comm.rank, self.comm.world, self.n_labels, self.lo,
                                                         self.hi, self.dim):
                raise ConfigError("shard checkpoint layout does not match this engine")
            if bool(bf16) != (self.W.dtype == torch.bfloat16) or bool(adam) != (self.optimizer == "adam"):
                raise ConfigError("shard checkpoint dtype / optimizer does not match this engine")
            rows = hi - lo
            wb = rows * dim * (2 if bf16 else 4)
            if fsize != hsize + wb + (2 * rows * dim * 4 if adam else 0):
                raise DataError("truncated or oversized shard checkpoint")  # nothing restored
            buf = fh.read(wb)
            if len(buf) != wb:
                raise DataError("truncated shard checkpoint")
            arr = np.frombuffer(buf, dtype=np.int16 if bf16 else np.float32).reshape(rows, dim)
            t = torch.from_numpy(arr.copy())
            self._w_version += 1
            self.W.copy_(t.view(torch.bfloat16) if bf16 else t)
            if adam:
                for dst in (self.m, self.v):
                    buf = fh.read(rows * dim * 4)
                    if len(buf) != rows * dim * 4:
                        raise DataError("truncated shard checkpoint")
                    dst.copy_(torch.from_numpy(np.frombuffer(buf, dtype=np.float32).reshape(rows, dim).copy()))
        self.adam_step = int(adam_step)
        self.w_absmax.fill_(float(w_absmax))
        # the refresh snapshot is not part of the file: drop any snapshot of the
        # previous weights (snapshot() rebuilds it from the restored W)
        self.snap_f32 = self.snap_bf16 = self.snap_f8 = None
        self.snapshot_epoch = int(snap)


class _HostPipe:
    """Double-buffered host->device staging on a copy stream plus a D2H stream.

    stage() copies a call's pinned inputs into device slot k (after the compute
    that last read slot k, tracked by release()) and makes the current stream
    wait for the copy; fetch() copies a result back on the D2H stream after the
    current stream's work. Slots are owned device buffers (never freed), so no
    caching-allocator reuse can race the side streams."""

    def __init__(self, device, n_slots: int = 2):
        self.device = device
        self.h2d = torch.cuda.Stream(device)
        self.d2h = torch.cuda.Stream(device)
        self.slots = [dict() for _ in range(n_slots)]
        self.free = [None] * n_slots
        self.k = 0

    def stage(self, tensors: dict):
        k = self.k
        self.k = (k + 1) % len(self.slots)
        bufs = self.slots[k]
        out = {}
        with torch.cuda.stream(self.h2d):
            if self.free[k] is not None:
                self.h2d.wait_event(self.free[k])
            for name, t in tensors.items():
                if t is None:
                    out[name] = None
                    continue
                n = t.numel()
                buf = bufs.get(name)
                if buf is None or buf.numel() < n or buf.dtype != t.dtype:
                    buf = torch.empty(max(n, 1), dtype=t.dtype, device=self.device)
                    bufs[name] = buf
                view = buf[:n].view(t.shape)
                view.copy_(t, non_blocking=True)
                out[name] = view
            ready = torch.cuda.Event()
            ready.record(self.h2d)
        torch.cuda.current_stream().wait_event(ready)
        return out, k

    def release(self, k: int) -> None:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.free[k] = ev

    def fetch(self, dev_tensor, host_out) -> None:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.d2h.wait_event(ev)
        with torch.cuda.stream(self.d2h):
            host_out.copy_(dev_tensor, non_blocking=True)
        dev_tensor.record_stream(self.d2h)


def _sum_in_rank_order(parts: torch.Tensor) -> torch.Tensor:
    """parts[0] + parts[1] + ... + parts[G-1], left to right (a fixed order,
    unlike a collective's reduction tree)."""
    acc = parts[0].clone()
    for r in range(1, parts.shape[0]):
        acc += parts[r]
    return acc


def h2d_bytes(*tensors) -> int:
    return int(sum(t.numel() * t.element_size() for t in tensors if t is not None))
