// topk.cuh — per-query running top-k for the refresh epilogues.
//
// Each query is owned by one thread (one TMEM lane in the tcgen05 kernel, one
// row of the score tile in the SIMT kernel). The thread admits a key only if
// it beats the current k-th best (tau), appending it to a small global buffer
// (L2-resident). When any lane's buffer could overflow, the WARP cooperatively
// compacts that lane's buffer: it drops the query's positives (the mask of
// anns.py:254-255), bitonic-sorts the keys descending and keeps k, which also
// raises tau. After warm-up admissions are rare (~k ln(n/k) per query), so
// the scan over scores is a compare per element and the scores never leave
// the SM.
#pragma once

#include "common.cuh"

namespace astra {

struct LaneTopK {
  uint64_t* buf;        // cap entries (this query's buffer)
  const int32_t* pos;   // this query's positives (sorted global ids)
  int64_t npos;
  int cnt;
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

// Warp-cooperative: filter positives out of buf[0:cnt], sort descending,
// keep the best k at buf[0:k]. Register bitonic network over P = 32*R slots.
// Returns the number of valid keys kept; *kth = k-th key if >= k valid else 0.
template <int R>
__device__ int compact_regs(uint64_t* buf, int cnt, const int32_t* pos, int64_t npos, int k, uint64_t* kth) {
  const int lane = threadIdx.x & 31;
  uint64_t x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int e = r * 32 + lane;
    uint64_t v = e < cnt ? buf[e] : 0ull;
    if (v && npos && sorted_contains(pos, npos, key_id(v))) v = 0ull;
    x[r] = v;
  }
  constexpr int P = 32 * R;
#pragma unroll
  for (int size = 2; size <= P; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int rs = stride >> 5;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if ((r & rs) == 0) {
            const int e = r * 32 + lane;
            const bool desc = (e & size) == 0;
            uint64_t a = x[r], b = x[r | rs];
            uint64_t hi = a > b ? a : b, lo = a > b ? b : a;
            x[r] = desc ? hi : lo;
            x[r | rs] = desc ? lo : hi;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int e = r * 32 + lane;
          const bool desc = (e & size) == 0;
          const bool lower = (lane & stride) == 0;
          uint64_t o = shfl_xor64(x[r], stride);
          uint64_t hi = x[r] > o ? x[r] : o, lo = x[r] > o ? o : x[r];
          x[r] = (lower == desc) ? hi : lo;
        }
      }
    }
  }
  int valid = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    valid += __popc(__ballot_sync(0xffffffffu, x[r] != 0ull));
    const int e = r * 32 + lane;
    if (e < k) buf[e] = x[r];
  }
  uint64_t kv = 0;
  if (valid >= k) {
    const int rk = (k - 1) >> 5, lk = (k - 1) & 31;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r == rk) kv = shfl64(x[r], lk);
  }
  *kth = kv;
  __syncwarp();
  return valid < k ? valid : k;
}

// Same contract for large buffers: bitonic network in (global) memory.
__device__ inline int compact_mem(uint64_t* buf, int cnt, int P, const int32_t* pos, int64_t npos, int k,
                                  uint64_t* kth) {
  const int lane = threadIdx.x & 31;
  int valid = 0;
  for (int e = lane; e < P; e += 32) {
    uint64_t v = e < cnt ? buf[e] : 0ull;
    if (v && npos && sorted_contains(pos, npos, key_id(v))) v = 0ull;
    buf[e] = v;
    valid += __popc(__ballot_sync(0xffffffffu, v != 0ull));
  }
  __syncwarp();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < P; i += 32) {
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

// Warp-uniform dispatch on the buffer capacity.
__device__ __forceinline__ int compact_any(uint64_t* buf, int cnt, int cap, const int32_t* pos, int64_t npos,
                                           int k, uint64_t* kth) {
  switch (cap) {
    case 64: return compact_regs<2>(buf, cnt, pos, npos, k, kth);
    case 128: return compact_regs<4>(buf, cnt, pos, npos, k, kth);
    case 256: return compact_regs<8>(buf, cnt, pos, npos, k, kth);
    case 512: return compact_regs<16>(buf, cnt, pos, npos, k, kth);
    default: return compact_mem(buf, cnt, cap, pos, npos, k, kth);
  }
}

// All 32 lanes call this before offering up to `incoming` keys each: every
// lane whose buffer could overflow is compacted by the whole warp.
__device__ __forceinline__ void topk_reserve(LaneTopK& t, int incoming, int cap, int k, bool active) {
  unsigned need = __ballot_sync(0xffffffffu, active && t.cnt + incoming > cap);
  const int lane = threadIdx.x & 31;
  while (need) {
    const int L = __ffs(need) - 1;
    need &= need - 1;
    uint64_t* b = reinterpret_cast<uint64_t*>(shfl64(reinterpret_cast<uint64_t>(t.buf), L));
    const int32_t* p = reinterpret_cast<const int32_t*>(shfl64(reinterpret_cast<uint64_t>(t.pos), L));
    const int64_t np = static_cast<int64_t>(shfl64(static_cast<uint64_t>(t.npos), L));
    const int c = __shfl_sync(0xffffffffu, t.cnt, L);
    uint64_t kth;
    int kept = compact_any(b, c, cap, p, np, k, &kth);
    if (lane == L) {
      t.cnt = kept;
      if (kth > t.tau) {
        t.tau = kth;
        t.tau_s = key_score(kth);
        if (t.gtau) atomicMax(reinterpret_cast<unsigned long long*>(t.gtau), static_cast<unsigned long long>(kth));
      }
    }
  }
}

// Final flush of every active lane: top-k keys (descending, zero-padded) to out[lane's row].
__device__ __forceinline__ void topk_flush(LaneTopK& t, int cap, int k, bool active, uint64_t* out_row) {
  unsigned act = __ballot_sync(0xffffffffu, active);
  const int lane = threadIdx.x & 31;
  while (act) {
    const int L = __ffs(act) - 1;
    act &= act - 1;
    uint64_t* b = reinterpret_cast<uint64_t*>(shfl64(reinterpret_cast<uint64_t>(t.buf), L));
    const int32_t* p = reinterpret_cast<const int32_t*>(shfl64(reinterpret_cast<uint64_t>(t.pos), L));
    const int64_t np = static_cast<int64_t>(shfl64(static_cast<uint64_t>(t.npos), L));
    const int c = __shfl_sync(0xffffffffu, t.cnt, L);
    uint64_t* o = reinterpret_cast<uint64_t*>(shfl64(reinterpret_cast<uint64_t>(out_row), L));
    uint64_t kth;
    int kept = compact_any(b, c, cap, p, np, k, &kth);
    for (int e = lane; e < k; e += 32) o[e] = e < kept ? b[e] : 0ull;
    __syncwarp();
  }
}

// Capacity for a given k: power of two with at least 64 free slots above k.
__host__ __device__ inline int topk_cap(int k) {
  int c = 64;
  while (c < 2 * k || c - k < 64) c <<= 1;
  return c;
}

}  // namespace astra
