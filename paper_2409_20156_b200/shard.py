"""Label-range sharding over torch.distributed (NCCL over NVLink on B200).

GPU g of G owns labels [lo_g, hi_g) of W and of its optimizer state
(data-parallel encoder, label-sharded classifier).
The collectives of one classifier step are:
  refresh  all_gather(queries, positives) -> local top-k per shard ->
           all_to_all(partial keys, by query owner) -> exact merge
           (astra_topk_merge) of the world partial lists of the rank's rows
  sample   all_gather(rows, positives, hard-cache rows) -> every shard runs
           the Philox sampler over all rows (keyed by global row id, so the
           slates are identical on every rank and to a 1-GPU run)
  step     all_gather(embeddings) -> shard-local loss/update ->
           reduce_scatter(grad_emb) to the data-parallel owners,
           all_reduce(loss partial, fp64)
W itself is never communicated. With world_size 1 every helper is the
identity and no collective is issued.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_labels: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous label range of `rank`: sizes differ by at most one."""
    base, extra = divmod(n_labels, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class Comm:
    """The few collectives the hot path needs; identity when world_size == 1."""

    def __init__(self, group=None):
        self.group = group
        self.enabled = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.enabled else 1
        self.rank = dist.get_rank(group) if self.enabled else 0
        # the tensor forms (all_gather_into_tensor, reduce_scatter_tensor,
        # all_to_all_single) run on NCCL and on gloo alike, so the CPU
        # world_size-2 tests exercise the same calls as the GPU path
        self.backend = dist.get_backend(group) if self.enabled else None

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """Concatenate equal-shaped tensors of all ranks along dim 0."""
        if self.world == 1:
            return t
        t = t.contiguous()
        out = torch.empty((self.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out

    def all_gather_stack(self, t: torch.Tensor) -> torch.Tensor:
        """[world, *t.shape] stack of every rank's tensor."""
        return self.all_gather(t.unsqueeze(0))

    def all_gather_ragged(self, t: torch.Tensor) -> tuple[torch.Tensor, list[int]]:
        """Concatenate 1-D tensors of different lengths; returns (cat, lengths)."""
        if self.world == 1:
            return t, [t.shape[0]]
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        lens = self.all_gather(n).tolist()
        m = max(lens)
        pad = torch.zeros(m, dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        g = self.all_gather(pad).view(self.world, m)
        return torch.cat([g[r, : lens[r]] for r in range(self.world)]), lens

    def reduce_scatter(self, t: torch.Tensor) -> torch.Tensor:
        """Sum over ranks, then keep this rank's dim-0 slice."""
        if self.world == 1:
            return t
        t = t.contiguous()
        out = torch.empty((t.shape[0] // self.world,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.reduce_scatter_tensor(out, t, group=self.group)
        return out

    def all_to_all(self, t: torch.Tensor) -> torch.Tensor:
        """Dim-0 chunk j of `t` goes to rank j; returns [world, n/world, ...]
        with chunk i received from rank i."""
        if self.world == 1:
            return t.unsqueeze(0)
        t = t.contiguous()
        out = torch.empty_like(t)
        dist.all_to_all_single(out, t, group=self.group)
        return out.view((self.world, t.shape[0] // self.world) + tuple(t.shape[1:]))

    def all_reduce(self, t: torch.Tensor, op: str = "sum") -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, op={"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}[op],
                            group=self.group)
        return t

    def barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)


def gather_csr(comm: Comm, indptr: torch.Tensor, ids: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """All-gather per-row CSR lists (e.g. positives) of every rank's rows."""
    if comm.world == 1:
        return indptr, ids
    counts = indptr[1:] - indptr[:-1]
    all_counts = comm.all_gather(counts)
    all_ids, _ = comm.all_gather_ragged(ids)
    out = torch.zeros(all_counts.shape[0] + 1, dtype=torch.int64, device=indptr.device)
    out[1:] = torch.cumsum(all_counts, 0)
    return out, all_ids
