// topk.cuh — per-query running top-k for the refresh epilogues.
//
// Each query is owned by one thread (one TMEM lane in the tcgen05 kernel, one
// row of the score tile in the SIMT kernel). The thread admits a key only if
// it beats the current k-th best (tau), appending it to a small global buffer
// (L2-resident). The buffer holds a sorted prefix (the best <= k keys so far)
// followed by up to P unsorted newcomers (P = next_pow2(k), capacity 2P).
// When a lane's newcomers could overflow, the WARP compacts that lane's
// buffer cooperatively: newcomers drop the query's positives (the mask of
// anns.py:254-255), get bitonic-sorted in registers and merged with the sorted
// prefix (max(A[i], B[P-1-i]) + one half-cleaner), which also raises tau.
// Keys are unique (distinct ids), so "key > tau" is exact. After warm-up
// admissions are rare (~k ln(n/k) per query) and the scan over scores is a
// compare per element: the scores never leave the SM.
#pragma once

#include "common.cuh"

namespace astra {

struct LaneTopK {
  uint64_t* buf;        // 2P entries: [0, nsorted) sorted desc, [nsorted, cnt) newcomers
  const int32_t* pos;   // this query's positives (sorted global ids)
  int64_t npos;
  int cnt, nsorted;
  uint64_t tau;         // admit keys > tau (0 = admit all)
  float tau_s;          // key_score(tau) or -inf: cheap score prefilter
  uint64_t* gtau;       // this query's threshold shared by every label partition (or null)
};

__device__ __forceinline__ void lane_init(LaneTopK& t, uint64_t* buf, const int32_t* pos, int64_t npos,
                                          uint64_t* gtau = nullptr) {
  t.buf = buf;
  t.pos = pos;
  t.npos = npos;
  t.cnt = 0;
  t.nsorted = 0;
  t.tau = 0;
  t.tau_s = -INFINITY;
  t.gtau = gtau;
}

// Raise tau to the query's shared threshold. Any partition's k-th best key is a
// valid bound for all of them: a key below it cannot be in the global top-k.
__device__ __forceinline__ void lane_sync_tau(LaneTopK& t) {
  if (t.gtau) {
    const uint64_t g = *reinterpret_cast<volatile uint64_t*>(t.gtau);
    if (g > t.tau) {
      t.tau = g;
      t.tau_s = key_score(g);
    }
  }
}

// Admit one candidate (caller guarantees room: see topk_reserve).
__device__ __forceinline__ void lane_offer(LaneTopK& t, float s, uint32_t gid) {
  if (s >= t.tau_s) {
    uint64_t key = make_key(s, gid);
    if (key > t.tau) t.buf[t.cnt++] = key;
  }
}

// Admit a pre-built key (merge of partial lists).
__device__ __forceinline__ void lane_offer_key(LaneTopK& t, uint64_t key) {
  if (key > t.tau) t.buf[t.cnt++] = key;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  uint32_t lo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v), src);
  uint32_t hi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), src);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int m) {
  uint32_t lo = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(v), m);
  uint32_t hi = __shfl_xor_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), m);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ uint64_t kmax(uint64_t a, uint64_t b) { return a > b ? a : b; }
__device__ __forceinline__ uint64_t kmin(uint64_t a, uint64_t b) { return a > b ? b : a; }

// Descending half-cleaner network on a bitonic sequence held as x[r] = element r*32+lane.
template <int R>
__device__ __forceinline__ void bitonic_clean_desc(uint64_t (&x)[R], int lane) {
#pragma unroll
  for (int stride = 16 * R; stride > 0; stride >>= 1) {
    if (stride >= 32) {
      const int rs = stride >> 5;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((r & rs) == 0) {
          const uint64_t a = x[r], b = x[r | rs];
          x[r] = kmax(a, b);
          x[r | rs] = kmin(a, b);
        }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint64_t o = shfl_xor64(x[r], stride);
        x[r] = ((lane & stride) == 0) ? kmax(x[r], o) : kmin(x[r], o);
      }
    }
  }
}

// Full descending bitonic sort of 32*R elements (x[r] = element r*32+lane).
template <int R>
__device__ __forceinline__ void bitonic_sort_desc(uint64_t (&x)[R], int lane) {
  constexpr int P = 32 * R;
#pragma unroll
  for (int size = 2; size <= P; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int rs = stride >> 5;
#pragma unroll
        for (int r = 0; r < R; ++r)
          if ((r & rs) == 0) {
            const bool desc = ((r * 32 + lane) & size) == 0;
            const uint64_t a = x[r], b = x[r | rs];
            x[r] = desc ? kmax(a, b) : kmin(a, b);
            x[r | rs] = desc ? kmin(a, b) : kmax(a, b);
          }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool desc = ((r * 32 + lane) & size) == 0;
          const bool lower = (lane & stride) == 0;
          const uint64_t o = shfl_xor64(x[r], stride);
          x[r] = (lower == desc) ? kmax(x[r], o) : kmin(x[r], o);
        }
      }
    }
  }
}

// Zero the keys of x[] whose id is one of the query's positives (the mask of
// anns.py:254-255). Up to 64 positives are held in two registers per lane and
// broadcast: one parallel load instead of a dependent binary search in global
// memory per key (which made compaction latency-bound).
template <int R>
__device__ __forceinline__ void drop_positives(uint64_t (&x)[R], const int32_t* pos, int64_t npos, int lane) {
  if (npos <= 0) return;
  if (npos <= 64) {
    const int32_t p0 = lane < npos ? pos[lane] : -1;
    const int32_t p1 = lane + 32 < npos ? pos[lane + 32] : -1;
    int32_t id[R];
    bool hit[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      id[r] = x[r] ? key_id(x[r]) : -2;
      hit[r] = false;
    }
    const int n = static_cast<int>(npos);
    for (int i = 0; i < n; ++i) {
      const int32_t pv = __shfl_sync(0xffffffffu, i < 32 ? p0 : p1, i & 31);
#pragma unroll
      for (int r = 0; r < R; ++r) hit[r] |= id[r] == pv;
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (hit[r]) x[r] = 0ull;
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (x[r] && sorted_contains(pos, npos, key_id(x[r]))) x[r] = 0ull;
  }
}

// Warp-cooperative compaction of one lane's buffer (P = 32*R): newcomers
// buf[ns, cnt) lose positives and are sorted; merged with the sorted prefix
// buf[0, ns) into the best k at buf[0, kept). Returns kept; *kth = k-th key
// when k valid keys exist, else 0.
template <int R>
__device__ int compact_regs(uint64_t* buf, int ns, int cnt, const int32_t* pos, int64_t npos, int k,
                            uint64_t* kth) {
  const int lane = threadIdx.x & 31;
  uint64_t nw[R], old[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = r * 32 + lane;
    nw[r] = ns + e < cnt ? buf[ns + e] : 0ull;
    old[r] = e < ns ? buf[e] : 0ull;
  }
  drop_positives<R>(nw, pos, npos, lane);
  bitonic_sort_desc<R>(nw, lane);
  // top P of (old u new): max(old[i], new[P-1-i]) is bitonic; clean it
#pragma unroll
  for (int r = 0; r < R; ++r) old[r] = kmax(old[r], shfl64(nw[R - 1 - r], 31 - lane));
  bitonic_clean_desc<R>(old, lane);
  int valid = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    valid += __popc(__ballot_sync(0xffffffffu, old[r] != 0ull));
    const int e = r * 32 + lane;
    if (e < k) buf[e] = old[r];
  }
  uint64_t kv = 0;
  if (valid >= k) {
    const int rk = (k - 1) >> 5, lk = (k - 1) & 31;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r == rk) kv = shfl64(old[r], lk);
  }
  *kth = kv;
  __syncwarp();
  return valid < k ? valid : k;
}

// Same contract for large k: full bitonic network over the 2P buffer in memory.
__device__ inline int compact_mem(uint64_t* buf, int cnt, int cap, const int32_t* pos, int64_t npos, int k,
                                  uint64_t* kth) {
  const int lane = threadIdx.x & 31;
  int valid = 0;
  for (int e = lane; e < cap; e += 32) {
    uint64_t v = e < cnt ? buf[e] : 0ull;
    if (v && npos && sorted_contains(pos, npos, key_id(v))) v = 0ull;
    buf[e] = v;
    valid += __popc(__ballot_sync(0xffffffffu, v != 0ull));
  }
  __syncwarp();
  for (int size = 2; size <= cap; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < cap; i += 32) {
        int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          uint64_t a = buf[i], b = buf[j];
          if ((a < b) == desc) {
            buf[i] = b;
            buf[j] = a;
          }
        }
      }
      __syncwarp();
    }
  }
  *kth = valid >= k ? buf[k - 1] : 0ull;
  __syncwarp();
  return valid < k ? valid : k;
}

// Capacity for a given k: 2P, P = next power of two >= max(k + 32, 64): the
// sorted prefix (<= k) plus a newcomer region of P (compaction every ~P-k..P
// admissions; larger P = fewer, slightly longer compactions).
__host__ __device__ inline int topk_cap(int k) {
  int p = 64;
  while (p < k + 32) p <<= 1;
  return 2 * p;
}

// Warp-uniform dispatch on the buffer capacity.
__device__ __forceinline__ int compact_any(uint64_t* buf, int ns, int cnt, int cap, const int32_t* pos,
                                           int64_t npos, int k, uint64_t* kth) {
  // (newcomer count is at most P = cap/2 here)
  switch (cap) {
    case 64: return compact_regs<1>(buf, ns, cnt, pos, npos, k, kth);
    case 128: return compact_regs<2>(buf, ns, cnt, pos, npos, k, kth);
    case 256: return compact_regs<4>(buf, ns, cnt, pos, npos, k, kth);
    case 512: return compact_regs<8>(buf, ns, cnt, pos, npos, k, kth);
    case 1024: return compact_regs<16>(buf, ns, cnt, pos, npos, k, kth);
    default: return compact_mem(buf, cnt, cap, pos, npos, k, kth);
  }
}

struct CompactResult {
  uint64_t kth;  // new k-th best key (0 if fewer than k valid keys)
  int kept;      // sorted prefix length after the compaction
};

// Out-of-line body of compact_lane: the bitonic networks are large, and
// inlining them at every call site bloats the epilogue loops far past the
// instruction cache (the fast path must stay a few hundred instructions).
static __device__ __noinline__ CompactResult compact_lane_impl(uint64_t* b, const int32_t* p, int64_t np, int c, int ns,
                                                        int cap, int k) {
  const int lane = threadIdx.x & 31;
  const int P = cap / 2;
  uint64_t kth = 0;
  int kept;
  while (true) {
    const int take = min(c - ns, P);
    const int rest = c - (ns + take);  // <= kTopkSlack: held in registers across the merge
    const uint64_t v0 = lane < rest ? b[ns + take + lane] : 0ull;
    const uint64_t v1 = lane + 32 < rest ? b[ns + take + 32 + lane] : 0ull;
    __syncwarp();
    uint64_t kk;
    kept = compact_any(b, ns, ns + take, cap, p, np, k, &kk);
    kth = kk > kth ? kk : kth;
    if (rest <= 0) break;
    // slide the unmerged newcomers down behind the new sorted prefix
    if (lane < rest) b[kept + lane] = v0;
    if (lane + 32 < rest) b[kept + 32 + lane] = v1;
    __syncwarp();
    ns = kept;
    c = kept + rest;
  }
  return CompactResult{kth, kept};
}

// Compact lane L's buffer (all 32 lanes participate). Newcomers beyond P are
// merged in further rounds (topk_settle lets up to kTopkSlack extra keys in).
__device__ __forceinline__ void compact_lane(LaneTopK& t, int L, int cap, int k) {
  const int lane = threadIdx.x & 31;
  uint64_t* b = reinterpret_cast<uint64_t*>(shfl64(reinterpret_cast<uint64_t>(t.buf), L));
  const int32_t* p = reinterpret_cast<const int32_t*>(shfl64(reinterpret_cast<uint64_t>(t.pos), L));
  const int64_t np = static_cast<int64_t>(shfl64(static_cast<uint64_t>(t.npos), L));
  const int c = __shfl_sync(0xffffffffu, t.cnt, L);
  const int ns = __shfl_sync(0xffffffffu, t.nsorted, L);
  const CompactResult r = compact_lane_impl(b, p, np, c, ns, cap, k);
  if (lane == L) {
    t.cnt = t.nsorted = r.kept;
    if (r.kth > t.tau) {
      t.tau = r.kth;
      t.tau_s = key_score(r.kth);
      if (t.gtau) atomicMax(reinterpret_cast<unsigned long long*>(t.gtau), static_cast<unsigned long long>(r.kth));
    }
  }
}

// Extra buffer entries beyond the logical capacity 2P: lets a lane append up
// to kTopkSlack keys before topk_settle() runs (allocate cap + kTopkSlack).
constexpr int kTopkSlack = 64;

// After unchecked offers of at most kTopkSlack keys per lane: compact every
// lane whose newcomer region exceeds P.
__device__ __forceinline__ void topk_settle(LaneTopK& t, int cap, int k, bool active) {
  unsigned need = __ballot_sync(0xffffffffu, active && (t.cnt - t.nsorted) > cap / 2);
  while (need) {
    const int L = __ffs(need) - 1;
    need &= need - 1;
    compact_lane(t, L, cap, k);
  }
}

// All 32 lanes call this before offering up to `incoming` keys each: every
// lane whose newcomer region could overflow is compacted by the whole warp.
__device__ __forceinline__ void topk_reserve(LaneTopK& t, int incoming, int cap, int k, bool active) {
  unsigned need = __ballot_sync(0xffffffffu, active && (t.cnt - t.nsorted) + incoming > cap / 2);
  while (need) {
    const int L = __ffs(need) - 1;
    need &= need - 1;
    compact_lane(t, L, cap, k);
  }
}

// Final flush of every active lane: top-k keys (descending, zero-padded) to out[lane's row].
__device__ __forceinline__ void topk_flush(LaneTopK& t, int cap, int k, bool active, uint64_t* out_row) {
  unsigned act = __ballot_sync(0xffffffffu, active);
  const int lane = threadIdx.x & 31;
  while (act) {
    const int L = __ffs(act) - 1;
    act &= act - 1;
    compact_lane(t, L, cap, k);
    uint64_t* b = reinterpret_cast<uint64_t*>(shfl64(reinterpret_cast<uint64_t>(t.buf), L));
    uint64_t* o = reinterpret_cast<uint64_t*>(shfl64(reinterpret_cast<uint64_t>(out_row), L));
    const int kept = __shfl_sync(0xffffffffu, t.cnt, L);
    for (int e = lane; e < k; e += 32) o[e] = e < kept ? b[e] : 0ull;
    __syncwarp();
  }
}

}  // namespace astra
