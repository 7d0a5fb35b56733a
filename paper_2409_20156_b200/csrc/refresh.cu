// refresh.cu — shortlist refresh orchestration, the fp32-exact SIMT path,
// cross-partition merge and the fp32 re-rank.
//
// Replaces the exact branch of retrieve_hard_negatives (anns.py:233-256):
// scores = E @ W^T (anns.py:253), positives masked (anns.py:254-255), top-k
// by (score desc, id asc) (anns.py:112-133). The score matrix is never
// materialised: each CTA streams a label range for a 128-query tile and keeps
// per-query running top-k lists (topk.cuh).
//
// Modes (include/astra_b200.h):
//   FP32_EXACT  SIMT FFMA tile kernel here; every score is the sequential
//               fmaf chain over t = 0..d-1, so ids are bit-identical to
//               oracle_refresh_fp32.
//   BF16        tcgen05 kernel (refresh_tc.cu), bf16 operands, fp32 accum.
//   BF16_RERANK tcgen05 top-k' (k' = max(1.5k, k+16)) then the k' candidates
//               are re-scored with the same sequential fmaf chain and
//               re-ranked: equal to FP32_EXACT whenever the exact top-k lies
//               inside the top-k'.
//   FP8_RERANK  the same pipeline on e4m3 operands (kind::f8f6f4, twice the
//               tensor rate): queries quantised per row here, labels from the
//               caller's e4m3 snapshot (astra_quantize_e4m3, one global
//               scale); a per-query / global scale does not change a query's
//               ranking. k' = max(2k, k+32) for the coarser candidate scores.
#include <cuda_fp8.h>
#include <math.h>

#include <vector>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"
#include "refresh_tc.cuh"
#include "topk.cuh"

namespace astra {


namespace {

constexpr int kBM = 128, kBN = 128, kBK = 8;
constexpr int kSimtThreads = 256;

// ------------------------------------------------------------- fp32 SIMT

struct SimtArgs {
  const float* Q;
  const float* W;
  int64_t nq, L, off;
  int d, k, cap, n_parts;
  int64_t labels_per_part;
  const int64_t* pos_indptr;
  const int32_t* pos_ids;
  uint64_t* bufs;       // [n_qtiles * n_parts * 128][cap]
  uint64_t* part_keys;  // [n_parts][nq][k]
  uint64_t* gtau;       // [nq] shared per-query thresholds
};

constexpr size_t kSimtSmem = sizeof(float) * (2 * kBK * kBM + 2 * kBK * kBN + kBM * (kBN + 1));

__global__ void __launch_bounds__(kSimtThreads) refresh_simt_kernel(SimtArgs a) {
  extern __shared__ __align__(16) float dsm[];
  float(*As)[kBK][kBM] = reinterpret_cast<float(*)[kBK][kBM]>(dsm);
  float(*Bs)[kBK][kBN] = reinterpret_cast<float(*)[kBK][kBN]>(dsm + 2 * kBK * kBM);
  float(*sc)[kBN + 1] = reinterpret_cast<float(*)[kBN + 1]>(dsm + 2 * kBK * kBM + 2 * kBK * kBN);
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int qt = blockIdx.x, part = blockIdx.y;
  const int64_t q0 = static_cast<int64_t>(qt) * kBM;
  const int64_t l_begin = static_cast<int64_t>(part) * a.labels_per_part;
  const int64_t l_end = std::min<int64_t>(a.L, l_begin + a.labels_per_part);

  // epilogue lane state (threads 0..127 own query rows)
  LaneTopK t;
  const bool row_owner = tid < kBM;
  const int64_t q = q0 + tid;
  const bool active = row_owner && q < a.nq;
  if (row_owner) {
    uint64_t* buf = a.bufs + ((static_cast<size_t>(qt) * a.n_parts + part) * kBM + tid) * (a.cap + kTopkSlack);
    const int64_t p0 = active ? a.pos_indptr[q] : 0, p1 = active ? a.pos_indptr[q + 1] : 0;
    lane_init(t, buf, a.pos_ids + p0, p1 - p0, active ? a.gtau + q : nullptr);
  }

  // loader mapping: 128 rows x 8 k per tile = 1024 floats, 4 per thread
  const int lrow = tid >> 1, lk = (tid & 1) * 4;
  for (int64_t lt = l_begin; lt < l_end; lt += kBN) {
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
    const int nkt = (a.d + kBK - 1) / kBK;
    auto load = [&](int kt, int buf) {
      const int kk = kt * kBK + lk;
      const int64_t qr = q0 + lrow, lr = lt + lrow;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kc = kk + u;
        As[buf][lk + u][lrow] = (qr < a.nq && kc < a.d) ? a.Q[qr * a.d + kc] : 0.0f;
        Bs[buf][lk + u][lrow] = (lr < l_end && kc < a.d) ? a.W[lr * a.d + kc] : 0.0f;
      }
    };
    load(0, 0);
    __syncthreads();
    for (int kt = 0; kt < nkt; ++kt) {
      const int cur = kt & 1;
      if (kt + 1 < nkt) load(kt + 1, cur ^ 1);
#pragma unroll
      for (int kk = 0; kk < kBK; ++kk) {
        float av[8], bv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = As[cur][kk][ty * 8 + i];
#pragma unroll
        for (int j = 0; j < 8; ++j) bv[j] = Bs[cur][kk][tx * 8 + j];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) sc[ty * 8 + i][tx * 8 + j] = acc[i][j];
    __syncthreads();
    if (row_owner) {
      lane_sync_tau(t);
      const int nl = static_cast<int>(std::min<int64_t>(kBN, l_end - lt));
      for (int c0 = 0; c0 < kBN; c0 += 32) {
        topk_reserve(t, 32, a.cap, a.k, active);
        if (active) {
          const int cn = std::min(32, nl - c0);
          for (int c = 0; c < cn; ++c)
            lane_offer(t, sc[tid][c0 + c], static_cast<uint32_t>(lt + c0 + c + a.off));
        }
      }
    }
    __syncthreads();
  }
  if (row_owner) {
    uint64_t* out = a.part_keys + (static_cast<size_t>(part) * a.nq + (active ? q : 0)) * a.k;
    topk_flush(t, a.cap, a.k, active, out);
  }
}

// ------------------------------------------------------------- merge

// One thread per query: offer the n_parts partial lists (layout [part][nq][k_in])
// and keep the best k_out. Keys already exclude positives.
__global__ void __launch_bounds__(128) merge_kernel(const uint64_t* part_keys, int64_t nq, int n_parts, int k_in,
                                                    int k_out, int cap, uint64_t* bufs, uint64_t* out_keys,
                                                    int32_t* out_ids, float* out_scores) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * 128 + threadIdx.x;
  const bool active = q < nq;
  LaneTopK t;
  lane_init(t, bufs + static_cast<size_t>(active ? q : 0) * (cap + kTopkSlack), nullptr, 0);
  for (int p = 0; p < n_parts; ++p) {
    const uint64_t* src = part_keys + (static_cast<size_t>(p) * nq + (active ? q : 0)) * k_in;
    for (int c0 = 0; c0 < k_in; c0 += 32) {
      topk_reserve(t, 32, cap, k_out, active);
      if (active) {
        const int cn = std::min(32, k_in - c0);
        for (int c = 0; c < cn; ++c) {
          uint64_t key = src[c0 + c];
          if (key) lane_offer_key(t, key);
        }
      }
    }
  }
  // flush into the buffer itself (rows are private), then decode
  topk_flush(t, cap, k_out, active, t.buf);
  if (active) {
    for (int j = 0; j < k_out; ++j) {
      uint64_t key = t.buf[j];
      if (out_keys) out_keys[q * k_out + j] = key;
      if (out_ids) out_ids[q * k_out + j] = key ? key_id(key) : -1;
      if (out_scores) out_scores[q * k_out + j] = key ? key_score(key) : -INFINITY;
    }
  }
}

// Warp per query: fold the n_parts descending-sorted partial lists into the
// running top-P (P = 32*R >= k_out). For two descending lists A, B the sequence
// max(A[i], B[P-1-i]) holds exactly the top P of A u B and is bitonic, so one
// half-cleaner pass re-sorts it. Exact, and independent of the part order.
template <int R>
__global__ void __launch_bounds__(256) merge_warp_kernel(const uint64_t* part_keys, int64_t nq, int n_parts,
                                                         int k_in, int k_out, uint64_t* out_keys, int32_t* out_ids,
                                                         float* out_scores, const int32_t* only,
                                                         const int32_t* qmap = nullptr,
                                                         const int32_t* n_active = nullptr) {
  constexpr int P = 32 * R;
  const int lane = threadIdx.x & 31;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (q >= nq) return;  // warp-uniform
  if (only && !only[q]) return;
  if (n_active && q >= *n_active) return;  // (compact verify: rows past the gathered ones)
  const int kin = k_in < P ? k_in : P;
  uint64_t cur[R];
  {
    const uint64_t* src = part_keys + static_cast<size_t>(q) * k_in;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = r * 32 + lane;
      cur[r] = e < kin ? src[e] : 0ull;
    }
  }
  for (int p = 1; p < n_parts; ++p) {
    const uint64_t* src = part_keys + (static_cast<size_t>(p) * nq + q) * k_in;
    uint64_t nx[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = r * 32 + lane;
      nx[r] = e < kin ? src[e] : 0ull;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint64_t o = shfl64(nx[R - 1 - r], 31 - lane);
      cur[r] = cur[r] > o ? cur[r] : o;
    }
#pragma unroll
    for (int stride = P / 2; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int rs = stride >> 5;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if ((r & rs) == 0) {
            const uint64_t a = cur[r], b = cur[r | rs];
            cur[r] = a > b ? a : b;
            cur[r | rs] = a > b ? b : a;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint64_t o = shfl_xor64(cur[r], stride);
          const bool lower = (lane & stride) == 0;
          cur[r] = lower ? (cur[r] > o ? cur[r] : o) : (cur[r] > o ? o : cur[r]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = r * 32 + lane;
    if (e < k_out) {
      const uint64_t key = cur[r];
      const size_t o = static_cast<size_t>(qmap ? qmap[q] : q) * k_out + e;
      if (out_keys) out_keys[o] = key;
      if (out_ids) out_ids[o] = key ? key_id(key) : -1;
      if (out_scores) out_scores[o] = key ? key_score(key) : -INFINITY;
    }
  }
}

// Compact verify: qmap[0..n) = the flagged queries in ascending order, *n_out =
// n (one CTA: a block-wide scan of the flags, 1024 at a time).
__global__ void __launch_bounds__(1024) compact_flagged_kernel(const int32_t* flags, int64_t nq, int32_t* qmap,
                                                               int32_t* n_out) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t i0 = 0; i0 < nq; i0 += 1024) {
    const int64_t i = i0 + threadIdx.x;
    const int f = i < nq && flags[i] ? 1 : 0;
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[warp] = __popc(b);
    __syncthreads();
    int before = base;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    if (f) qmap[before + __popc(b & ((1u << lane) - 1u))] = static_cast<int32_t>(i);
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < 32; ++w) t += wsum[w];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = base;
}

// Gather the flagged queries' tensor-core rows (row_bytes each, 16 B aligned)
// to the front of dst: block per row slot.
__global__ void __launch_bounds__(128) gather_rows_kernel(const unsigned char* src, int64_t row_bytes,
                                                          const int32_t* qmap, const int32_t* n_active,
                                                          unsigned char* dst) {
  const int64_t r = blockIdx.x;
  if (r >= *n_active) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<int64_t>(qmap[r]) * row_bytes);
  uint4* t = reinterpret_cast<uint4*>(dst + r * row_bytes);
  for (int64_t i = threadIdx.x; i < row_bytes / 16; i += blockDim.x) t[i] = s[i];
}

// ------------------------------------------------------------- fp32 re-rank

// Block per query (4 warps): re-score the k' candidates with the sequential
// fmaf chain (the FP32_EXACT order), sort the keys descending in shared memory,
// keep k. Each warp owns 32 candidates at a time and stages their rows through
// shared memory 64 floats per step with coalesced 16 B loads (lane t then runs
// its candidate's chain from a padded row: conflict-free). Needs d % 64 == 0.
constexpr int kRrWarps = 4, kRrChunk = 64, kRrPitch = kRrChunk + 1;

__global__ void __launch_bounds__(kRrWarps * 32) rerank_kernel(const float* Q, const float* W, int d, int64_t off,
                                                               const uint64_t* cand, int kc, int k,
                                                               uint64_t* out_keys, int32_t* out_ids,
                                                               float* out_scores) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t q = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int Pn = 1;
  while (Pn < kc) Pn <<= 1;
  float* qs = reinterpret_cast<float*>(smem);
  float* tile = qs + d + warp * 32 * kRrPitch;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem + align_up(sizeof(float) * (d + kRrWarps * 32 * kRrPitch), 16));
  for (int t = threadIdx.x; t < d; t += blockDim.x) qs[t] = Q[q * d + t];
  for (int c = threadIdx.x; c < Pn; c += blockDim.x) keys[c] = 0ull;
  __syncthreads();
  for (int c0 = warp * 32; c0 < kc; c0 += kRrWarps * 32) {
    const int c = c0 + lane;
    const uint64_t ck = c < kc ? cand[q * kc + c] : 0ull;
    const int32_t gid = ck ? key_id(ck) : -1;
    float s = 0.0f;
    for (int t0 = 0; t0 < d; t0 += kRrChunk) {
      // 32 rows x 64 floats: 2 rows per instruction, 16 lanes x 16 B each
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        const int r = 2 * i + (lane >> 4);
        const int32_t rg = __shfl_sync(0xffffffffu, gid, r);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (rg >= 0) v = __ldg(reinterpret_cast<const float4*>(W + static_cast<size_t>(rg - off) * d + t0) + (lane & 15));
        float* dst = tile + r * kRrPitch + (lane & 15) * 4;
        dst[0] = v.x;
        dst[1] = v.y;
        dst[2] = v.z;
        dst[3] = v.w;
      }
      __syncwarp();
      const float* row = tile + lane * kRrPitch;
#pragma unroll 16
      for (int t = 0; t < kRrChunk; ++t) s = fmaf(qs[t0 + t], row[t], s);
      __syncwarp();
    }
    if (ck) keys[c] = make_key(s, static_cast<uint32_t>(gid));
  }
  __syncthreads();
  for (int size = 2; size <= Pn; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < Pn; i += blockDim.x) {
        int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          uint64_t x = keys[i], z = keys[j];
          if ((x < z) == desc) {
            keys[i] = z;
            keys[j] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    uint64_t key = keys[j];
    if (out_keys) out_keys[q * k + j] = key;
    if (out_ids) out_ids[q * k + j] = key ? key_id(key) : -1;
    if (out_scores) out_scores[q * k + j] = key ? key_score(key) : -INFINITY;
  }
}

// TMA-fed re-rank (kc <= 512): CTA per query, a producer warp whose lanes
// bulk-copy their candidate's fp32 row, ch floats at a time, into a 2-stage
// ring (32 rows x ch floats, pitch 4 words mod 32: conflict-free LDS.128), and
// a consumer warp whose lane t runs candidate t's sequential fmaf chain over
// t = 0..d-1 (the FP32_EXACT order) across the chunks. Keys are sorted in
// registers (warp bitonic) and the best k written. 3 CTAs per SM keep ~200 KB
// of rows in flight per SM; the old kernel stalled on each 64-float chunk.
constexpr int kRtRing = 2;

__host__ __device__ inline int rerank_chunk(int d) { return d % 256 == 0 ? 256 : 64; }

template <int R, bool BF16>
__global__ void __launch_bounds__(64) rerank_tma_kernel(const float* Q, const void* W, int d, int64_t off,
                                                        const uint64_t* cand, int kc, int k, uint64_t* out_keys,
                                                        int32_t* out_ids, float* out_scores) {
  extern __shared__ __align__(128) unsigned char rsm[];
  const int ch = rerank_chunk(d);
  constexpr int esz = BF16 ? 2 : 4;
  const int pitch = ch * esz + 16;
  const int stage_bytes = 32 * pitch;
  unsigned char* ring = rsm;
  float* qs = reinterpret_cast<float*>(rsm + kRtRing * stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(qs + d);
  uint64_t* empty = full + kRtRing;
  const int64_t q = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = d / ch;
  const int n_units = (kc + 31) / 32;
  for (int t = threadIdx.x; t < d; t += 64) qs[t] = Q[q * d + t];
  if (threadIdx.x == 0) {
    for (int r = 0; r < kRtRing; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    // ---------------- producer: lane t copies candidate u*32+t's row chunks
    // (units of 32 empty keys — candidates filtered out by the caller — are
    // skipped by both warps; `seq` numbers the stage fills actually made)
    int seq = 0;
    for (int u = 0; u < n_units; ++u) {
      const int c = u * 32 + lane;
      const uint64_t key = c < kc ? cand[q * kc + c] : 0ull;
      const int32_t gid = key ? key_id(key) : -1;
      const unsigned live = __ballot_sync(0xffffffffu, gid >= 0);
      if (!live) continue;
      const uint32_t nbytes = __popc(live) * ch * esz;
      for (int h = 0; h < nch; ++h) {
        const int i = seq++, st = i % kRtRing;
        mbar_wait(&empty[st], ((i / kRtRing) & 1) ^ 1);
        if (lane == 0) mbar_expect_tx(&full[st], nbytes);
        __syncwarp();
        if (gid >= 0)
          bulk_g2s(ring + st * stage_bytes + lane * pitch,
                   static_cast<const unsigned char*>(W) + (static_cast<size_t>(gid - off) * d + h * ch) * esz,
                   ch * esz, &full[st]);
      }
    }
    return;
  }
  // ---------------- consumer
  uint64_t keys[R];
#pragma unroll
  for (int u = 0; u < R; ++u) keys[u] = 0ull;
  int seq = 0;
#pragma unroll
  for (int u = 0; u < R; ++u) {
    if (u < n_units) {
      const int c = u * 32 + lane;
      const uint64_t key = c < kc ? cand[q * kc + c] : 0ull;
      const int32_t gid = key ? key_id(key) : -1;
      if (!__ballot_sync(0xffffffffu, gid >= 0)) continue;
      float s = 0.0f;
      for (int h = 0; h < nch; ++h) {
        const int i = seq++, st = i % kRtRing;
        mbar_wait(&full[st], (i / kRtRing) & 1);
        const unsigned char* row = ring + st * stage_bytes + lane * pitch;
        const float* qh = qs + h * ch;
#pragma unroll 8
        for (int t = 0; t < ch; t += 4) {
          float4 v;
          if constexpr (BF16) {
            const uint2 u = *reinterpret_cast<const uint2*>(row + t * 2);
            v = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                            __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
          } else {
            v = *reinterpret_cast<const float4*>(row + t * 4);
          }
          const float4 x = *reinterpret_cast<const float4*>(qh + t);
          s = fmaf(x.x, v.x, s);
          s = fmaf(x.y, v.y, s);
          s = fmaf(x.z, v.z, s);
          s = fmaf(x.w, v.w, s);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      keys[u] = gid >= 0 ? make_key(s, static_cast<uint32_t>(gid)) : 0ull;
    }
  }
  bitonic_sort_desc<R>(keys, lane);
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const int e = u * 32 + lane;
    if (e < k) {
      const uint64_t key = keys[u];
      const size_t o = static_cast<size_t>(q) * k + e;
      if (out_keys) out_keys[o] = key;
      if (out_ids) out_ids[o] = key ? key_id(key) : -1;
      if (out_scores) out_scores[o] = key ? key_score(key) : -INFINITY;
    }
  }
}

template <int R, bool BF16>
int launch_rerank_tma(const float* qf, const void* wl, int d, int64_t off, const uint64_t* cand, int64_t nq, int kc,
                      int k, uint64_t* out_keys, int32_t* out_ids, float* out_scores, cudaStream_t st) {
  const int ch = rerank_chunk(d);
  const size_t smem = static_cast<size_t>(kRtRing) * 32 * (ch * (BF16 ? 2 : 4) + 16) + sizeof(float) * d + 16 * kRtRing;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rerank_tma_kernel<R, BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  rerank_tma_kernel<R, BF16><<<static_cast<unsigned>(nq), 64, smem, st>>>(qf, wl, d, off, cand, kc, k, out_keys,
                                                                          out_ids, out_scores);
  ASTRA_LAUNCHED("rerank_tma");
  return ASTRA_OK;
}

}  // namespace

// The fp32 re-rank on its own: score the caller's candidate keys (zero keys =
// none) against the fp32 (or bf16) label rows with the FP32_EXACT fmaf order
// and keep the best k (the multi-GPU refresh re-ranks only the candidates at
// or above the global k'-th bf16 key, engine.refresh).
int rerank_only(const float* qf, int64_t nq, int d, const uint64_t* cand, int kc, const void* labels, int w_dtype,
                int64_t off, int k, uint64_t* out_keys, int32_t* out_ids, float* out_scores, cudaStream_t st) {
  if (nq <= 0) return ASTRA_OK;
  if (k < 1 || k > kc) return set_error(ASTRA_ERR_CONFIG, "rerank: need 1 <= k <= kc (k=%d, kc=%d)", k, kc);
  const bool bf16 = w_dtype == ASTRA_W_BF16;
  if (kc <= 512 && d % 64 == 0 && (reinterpret_cast<uintptr_t>(labels) & 15) == 0) {
    auto go = [&](auto r_tag) {
      constexpr int R = decltype(r_tag)::value;
      return bf16 ? launch_rerank_tma<R, true>(qf, labels, d, off, cand, nq, kc, k, out_keys, out_ids, out_scores, st)
                  : launch_rerank_tma<R, false>(qf, labels, d, off, cand, nq, kc, k, out_keys, out_ids, out_scores, st);
    };
    if (kc <= 32) return go(std::integral_constant<int, 1>());
    if (kc <= 64) return go(std::integral_constant<int, 2>());
    if (kc <= 128) return go(std::integral_constant<int, 4>());
    if (kc <= 256) return go(std::integral_constant<int, 8>());
    return go(std::integral_constant<int, 16>());
  }
  if (bf16) return set_error(ASTRA_ERR_CONFIG, "rerank from bf16 labels needs kc <= 512, d %% 64 == 0");
  int Pn = 1;
  while (Pn < kc) Pn <<= 1;
  const size_t smem = align_up(sizeof(float) * (d + kRrWarps * 32 * kRrPitch), 16) + sizeof(uint64_t) * Pn;
  if (smem > 48 * 1024) cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  rerank_kernel<<<static_cast<unsigned>(nq), kRrWarps * 32, smem, st>>>(qf, static_cast<const float*>(labels), d, off,
                                                                         cand, kc, k, out_keys, out_ids, out_scores);
  ASTRA_LAUNCHED("rerank");
  return ASTRA_OK;
}

namespace {

__global__ void f32_to_bf16_kernel(const float* src, uint16_t* dst, int64_t n) {
  const int64_t i0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * 4;
  const bool aligned = (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 7) == 0;
  int64_t i = i0;
  if (aligned)  // two 16-byte loads in flight per thread
    for (; i + stride + 4 <= n; i += 2 * stride) {
      const float4 v0 = *reinterpret_cast<const float4*>(src + i);
      const float4 v1 = *reinterpret_cast<const float4*>(src + i + stride);
      uint2 o0, o1;
      o0.x = static_cast<uint32_t>(f32_to_bf16_bits(v0.x)) | (static_cast<uint32_t>(f32_to_bf16_bits(v0.y)) << 16);
      o0.y = static_cast<uint32_t>(f32_to_bf16_bits(v0.z)) | (static_cast<uint32_t>(f32_to_bf16_bits(v0.w)) << 16);
      o1.x = static_cast<uint32_t>(f32_to_bf16_bits(v1.x)) | (static_cast<uint32_t>(f32_to_bf16_bits(v1.y)) << 16);
      o1.y = static_cast<uint32_t>(f32_to_bf16_bits(v1.z)) | (static_cast<uint32_t>(f32_to_bf16_bits(v1.w)) << 16);
      *reinterpret_cast<uint2*>(dst + i) = o0;
      *reinterpret_cast<uint2*>(dst + i + stride) = o1;
    }
  for (; i < n; i += stride) {
    if (i + 4 <= n && (reinterpret_cast<uintptr_t>(src + i) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst + i) & 7) == 0) {
      float4 v = *reinterpret_cast<const float4*>(src + i);
      uint2 o;
      o.x = static_cast<uint32_t>(f32_to_bf16_bits(v.x)) | (static_cast<uint32_t>(f32_to_bf16_bits(v.y)) << 16);
      o.y = static_cast<uint32_t>(f32_to_bf16_bits(v.z)) | (static_cast<uint32_t>(f32_to_bf16_bits(v.w)) << 16);
      *reinterpret_cast<uint2*>(dst + i) = o;
    } else {
      for (int64_t j = i; j < n && j < i + 4; ++j) dst[j] = f32_to_bf16_bits(src[j]);
    }
  }
}

// ------------------------------------------------------------- e4m3 quantisation
__device__ __forceinline__ uint32_t e4m3x4(float a, float b, float c, float e) {
  const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
  const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(make_float2(c, e), __NV_SATFINITE, __NV_E4M3);
  return static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
}

// Query rows -> e4m3 with a per-row scale 448 / max|row| (warp per row,
// d % 128 == 0). The scale multiplies every score of the row alike, so the
// row's ranking is that of the unscaled products.
__global__ void quant_rows_e4m3_kernel(const float* __restrict__ src, int64_t rows, int d, uint8_t* __restrict__ dst) {
  const int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* x = src + r * d;
  float m = 0.0f;
  for (int t = lane * 4; t < d; t += 128) {
    const float4 v = *reinterpret_cast<const float4*>(x + t);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float sc = m > 0.0f && isfinite(m) ? 448.0f / m : 1.0f;
  for (int t = lane * 4; t < d; t += 128) {
    const float4 v = *reinterpret_cast<const float4*>(x + t);
    *reinterpret_cast<uint32_t*>(dst + r * d + t) = e4m3x4(v.x * sc, v.y * sc, v.z * sc, v.w * sc);
  }
}

template <bool BF16>
__device__ __forceinline__ float4 load4(const void* src, int64_t i) {
  if constexpr (BF16) {
    const uint2 u = *reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(src) + i);
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                       __uint_as_float(u.y & 0xFFFF0000u));
  } else {
    return *reinterpret_cast<const float4*>(static_cast<const float*>(src) + i);
  }
}

// max|x| over n values (n % 4 == 0) into scratch[0] (as bits; non-negative
// floats order as unsigned integers; a NaN reads as the largest)
template <bool BF16>
__global__ void absmax_kernel(const void* src, int64_t n, unsigned* out_bits) {
  float m = 0.0f;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * 4; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x * 4) {
    const float4 v = load4<BF16>(src, i);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits, __float_as_uint(m));
}

// x * scale -> e4m3, scale = 448 / max|x| read from scratch (1 when 0 or not finite)
template <bool BF16>
__global__ void quant_e4m3_kernel(const void* src, int64_t n, const unsigned* max_bits, float* scale_out,
                                  uint8_t* dst) {
  const float m = __uint_as_float(*max_bits);
  const float sc = m > 0.0f && isfinite(m) ? 448.0f / m : 1.0f;
  if (scale_out && blockIdx.x == 0 && threadIdx.x == 0) *scale_out = sc;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * 4; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x * 4) {
    const float4 v = load4<BF16>(src, i);
    *reinterpret_cast<uint32_t*>(dst + i) = e4m3x4(v.x * sc, v.y * sc, v.z * sc, v.w * sc);
  }
}

// ------------------------------------------------------------- select (two-pass refresh)

// The j-th largest of n 32-bit values (j >= 1, duplicates counted) by an
// MSB-first radix select with 8-bit digits: 4 passes over the values, each
// building a 256-bin histogram of the values matching the prefix so far in
// the warp's shared memory. get(i, &v) returns false for values to ignore.
template <class Get>
__device__ __forceinline__ uint32_t warp_kth_largest(Get get, int n, int j, uint32_t* hist, int lane) {
  uint32_t prefix = 0, mask = 0;
  int need = j;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0u;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      uint32_t x;
      if (get(i, x) && (x & mask) == prefix) atomicAdd(&hist[(x >> shift) & 255u], 1u);
    }
    __syncwarp();
    // lane l owns bins 255-8l .. 248-8l (descending); inclusive scan from the top
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      c[t] = hist[255 - 8 * lane - t];
      sum += c[t];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - sum;
    const unsigned owner = __ballot_sync(0xffffffffu, excl < static_cast<uint32_t>(need) &&
                                                          incl >= static_cast<uint32_t>(need));
    int digit = 0, before = 0;
    if (owner) {
      const int src = __ffs(owner) - 1;
      uint32_t cum = __shfl_sync(0xffffffffu, excl, src);
      int dd = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t ct = __shfl_sync(0xffffffffu, c[t], src);
        if (cum < static_cast<uint32_t>(need) && cum + ct >= static_cast<uint32_t>(need) && dd == 0) {
          digit = 255 - 8 * src - t;
          before = static_cast<int>(cum);
          dd = 1;
        }
        cum += ct;
      }
    } else {
      return 0u;  // fewer than j values
    }
    need -= before;
    prefix |= static_cast<uint32_t>(digit) << shift;
    mask |= 255u << shift;
    __syncwarp();
  }
  return prefix;
}

// Warp per query: the j-th largest of the query's 64-label group maxima
// (orderable bits, gmax [nq][n_groups]) by an MSB-first radix select. Each of
// the top-j group maxima is a distinct label, so at least j sampled labels
// score >= it: tau_keys[q] = (T << 32) admits every key with score >= T.
__global__ void __launch_bounds__(256) tau_select_kernel(const uint32_t* gmax, int64_t nq, int n_groups, int j,
                                                         uint64_t* tau_keys) {
  __shared__ uint32_t hist[8][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (q >= nq) return;  // warp-uniform
  const uint32_t* v = gmax + static_cast<size_t>(q) * n_groups;
  uint32_t T = 0;
  if (n_groups >= j)
    T = warp_kth_largest([&](int i, uint32_t& x) { x = __ldg(v + i); return true; }, n_groups, j, hist[warp], lane);
  if (lane == 0) tau_keys[q] = static_cast<uint64_t>(T) << 32;
}

// The label-sharded refresh's sample statistics: per query the j largest
// sampled group maxima of this shard (orderable bits, any order; ties at the
// j-th value filled in index order), from which the rows' owners take the
// global j-th largest over all shards.
__global__ void __launch_bounds__(256) sample_top_kernel(const uint32_t* gmax, int64_t nq, int n_groups, int j,
                                                         uint32_t* out) {
  __shared__ uint32_t hist[8][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (q >= nq) return;  // warp-uniform
  const uint32_t* v = gmax + static_cast<size_t>(q) * n_groups;
  uint32_t* o = out + static_cast<size_t>(q) * j;
  uint32_t T = 0;
  if (n_groups >= j)
    T = warp_kth_largest([&](int i, uint32_t& x) { x = __ldg(v + i); return true; }, n_groups, j, hist[warp], lane);
  int n = 0;
  for (int pass = 0; pass < 2 && n < j; ++pass) {  // values > T, then == T
    for (int i0 = 0; i0 < n_groups && n < j; i0 += 32) {
      const int i = i0 + lane;
      const uint32_t x = i < n_groups ? __ldg(v + i) : 0u;
      const bool take = i < n_groups && (pass == 0 ? x > T : x == T);
      const unsigned b = __ballot_sync(0xffffffffu, take);
      const int at = n + __popc(b & ((1u << lane) - 1u));
      if (take && at < j) o[at] = x;
      n += __popc(b);
    }
  }
  for (int e = n + lane; e < j; e += 32) o[e] = 0u;  // (fewer sampled groups than j)
}

// Warp per query: gather the FIXED-mode candidate lists of the query's label
// parts, drop the query's positives (anns.py:254-255) and keep the top k in
// (score desc, id asc) order: a radix select of the k-th largest score over
// the candidates, then a bitonic sort of the (usually exactly k) keys at or
// above it. The result is exact whenever at least k non-positive candidates
// exist and no list overflowed (every key of the true top-k is >= the k-th
// candidate >= the threshold, hence a candidate); otherwise the query is
// flagged for the exact running-top-k fallback.
constexpr int kSelWarps = 4, kSelSmall = 256, kSelPos = 128, kSelMaxParts = 64;

// Capacity of R, the keys at or above T2 (about k + |P| of them): a power of
// two >= max(kSelSmall, 2k).
inline int sel_rcap(int k) {
  int r = kSelSmall;
  while (r < 2 * k) r <<= 1;
  return r;
}

__global__ void __launch_bounds__(kSelWarps * 32) select_kernel(const uint64_t* cand, const int32_t* cand_cnt,
                                                                int n_parts, int cand_cap, int64_t nq,
                                                                const int64_t* pos_indptr, const int32_t* pos_ids,
                                                                int k, int sel_max, int rcap, uint64_t* out_keys,
                                                                int32_t* out_ids, float* out_scores, int32_t* flags,
                                                                int32_t* local_counts = nullptr) {
  // per warp: the candidates' 32-bit score parts (the radix select reads
  // them four times) and R, the full keys of those at or above T2 (read back
  // from the lists) — half the staging of full keys, so more warps per SM
  extern __shared__ __align__(16) uint64_t sel_smem[];
  __shared__ int32_t sel_off[kSelWarps][kSelMaxParts + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * kSelWarps + warp;
  if (q >= nq) return;  // warp-uniform
  uint64_t* R = sel_smem + static_cast<size_t>(warp) * (rcap + sel_max / 2);
  uint32_t* S = reinterpret_cast<uint32_t*>(R + rcap);
  // the parts' counts lane-parallel (up to kSelMaxParts = 64 parts: two per
  // lane), their offsets by a warp scan
  int total = 0;
  bool overflow = n_parts > kSelMaxParts;
  for (int pb = 0; pb < n_parts && !overflow; pb += 32) {
    const int p = pb + lane;
    const int c = p < n_parts ? cand_cnt[static_cast<size_t>(p) * nq + q] : 0;
    overflow |= __any_sync(0xffffffffu, c > cand_cap);
    const int cc = c < cand_cap ? c : cand_cap;
    int incl = cc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    if (p < n_parts) sel_off[warp][p] = total + incl - cc;
    total += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0 && !overflow) sel_off[warp][n_parts] = total;
  bool fail = overflow || total > sel_max;
  if (lane == 0 && fail) {
    flags[q] = 1;
    if (local_counts) local_counts[q] = 0;
  }
  if (fail) return;
  __syncwarp();
  const int64_t p0 = pos_indptr[q], np = pos_indptr[q + 1] - p0;
  // key of candidate i (parts concatenated in order). Each lane walks i
  // upwards in steps of 32, so its part index only moves forward: `pc` is the
  // lane's cursor (the last part whose offset is <= i; empty parts share their
  // successor's offset and are stepped over).
  auto key_at = [&](int i, int& pc) {
    while (pc + 1 < n_parts && sel_off[warp][pc + 1] <= i) ++pc;
    return cand[(static_cast<size_t>(pc) * nq + q) * cand_cap + (i - sel_off[warp][pc])];
  };
  // 1. the candidates' scores -> shared memory: few parts -> the warp walks
  //    each part (coalesced); many small parts (the SM-filling layouts) ->
  //    lane p copies part p (independent loads, no per-element part lookup)
  if (n_parts <= 4) {
    for (int p = 0; p < n_parts; ++p) {
      const int o = sel_off[warp][p], c = sel_off[warp][p + 1] - o;
      const uint64_t* src = cand + (static_cast<size_t>(p) * nq + q) * cand_cap;
#pragma unroll 4
      for (int e = lane; e < c; e += 32) S[o + e] = static_cast<uint32_t>(src[e] >> 32);
    }
  } else {
    for (int p = lane; p < n_parts; p += 32) {
      const int o = sel_off[warp][p], c = sel_off[warp][p + 1] - o;
      const uint64_t* src = cand + (static_cast<size_t>(p) * nq + q) * cand_cap;
#pragma unroll 4
      for (int e = 0; e < c; ++e) S[o + e] = static_cast<uint32_t>(src[e] >> 32);
    }
  }
  __syncwarp();
  // 2. T2 = the (k + |P|)-th largest score over ALL candidates: at most |P| of
  //    the keys above the k-th non-positive one are positives, so every key of
  //    the non-positive top k is >= T2 (0 when there are fewer candidates)
  __shared__ uint32_t sel_hist[kSelWarps][256];
  const int64_t k2l = static_cast<int64_t>(k) + np;
  const int k2 = static_cast<int>(k2l < total ? k2l : total);
  const uint32_t T = warp_kth_largest(
      [&](int i, uint32_t& x) {
        x = S[i];
        return true;
      },
      total, k2, sel_hist[warp], lane);
  // 3. warp-aggregated compaction of the keys with score >= T2 (full keys
  //    fetched back from the lists for those only)
  int nr = 0;
  int pc = 0;
  for (int i0 = 0; i0 < total; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t sc = i < total ? S[i] : 0u;
    const bool take = i < total && sc >= T;
    const unsigned bm = __ballot_sync(0xffffffffu, take);
    const int at = nr + __popc(bm & ((1u << lane) - 1u));
    if (take && at < rcap) {
      const uint64_t v = key_at(i, pc);
      R[at] = v;
    }
    nr += __popc(bm);
  }
  __syncwarp();
  if (nr > rcap) {  // pathological score ties: the exact fallback
    if (lane == 0) {
      flags[q] = 1;
      if (local_counts) local_counts[q] = 0;
    }
    return;
  }
  uint64_t* X = R;
  const int n = nr;
  // 4. drop the query's positives (anns.py:254-255) among them (positives in shared memory)
  __shared__ int32_t sel_pos[kSelWarps][kSelPos];
  const bool pos_smem = np <= kSelPos;
  if (pos_smem)
    for (int e = lane; e < np; e += 32) sel_pos[warp][e] = pos_ids[p0 + e];
  __syncwarp();
  const int32_t* Pp = pos_smem ? sel_pos[warp] : pos_ids + p0;
  int valid = 0;
  for (int e = lane; e < n; e += 32) {
    uint64_t v = X[e];
    if (v && np > 0 && sorted_contains(Pp, np, key_id(v))) X[e] = v = 0ull;
    valid += v != 0ull;
  }
  // local (label-sharded, global threshold): fewer than k here is normal —
  // the shards' counts decide globally which queries need the verify pass
  const int nvalid = warp_sum(valid);
  fail = !local_counts && nvalid < k;
  if (lane == 0) {
    flags[q] = fail ? 1 : 0;
    if (local_counts) local_counts[q] = nvalid < k ? nvalid : k;
  }
  if (fail) return;
  __syncwarp();
  int Pn = 1;
  while (Pn < n) Pn <<= 1;
  // zero-pad to the sort width and (local mode: fewer than k candidates is
  // normal) to the k keys written out; R holds rcap >= 2k entries
  for (int e = n + lane; e < (Pn > k ? Pn : k); e += 32) X[e] = 0ull;
  __syncwarp();
  for (int size = 2; size <= Pn; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (Pn >> 1); i += 32) {
        const int x = 2 * stride * (i / stride) + (i & (stride - 1));
        const int y = x + stride;
        const bool desc = (x & size) == 0;
        const uint64_t va = X[x], vb = X[y];
        if ((va < vb) == desc) {
          X[x] = vb;
          X[y] = va;
        }
      }
      __syncwarp();
    }
  }
  for (int jj = lane; jj < k; jj += 32) {
    const uint64_t key = X[jj];
    const size_t o = static_cast<size_t>(q) * k + jj;
    if (out_keys) out_keys[o] = key;
    if (out_ids) out_ids[o] = key_id(key);
    if (out_scores) out_scores[o] = key_score(key);
  }
}

// ------------------------------------------------------------- workspace

struct RefreshWs {
  uint64_t* gtau;
  void* qb;  // queries converted for the tensor cores: bf16, or e4m3 bytes (FP8_RERANK)
  uint64_t* bufs;
  uint64_t* part_keys;
  uint64_t* merge_bufs;
  uint64_t* rr_cand;    // BF16_RERANK: bf16 top-k' per query before the fp32 re-rank
  // two-pass (sample / threshold / select / verify)
  uint32_t* gmax;       // [nq][n_groups] group maxima of the label sample
  uint64_t* tau_keys;   // [nq] per-query threshold
  uint64_t* cand;       // [n_parts][nq][cand_cap]
  int32_t* cand_cnt;    // [n_parts][nq]
  int32_t* flags;       // [nq] 1 = select could not prove exactness -> fallback
  // compact verify
  void* qc;             // [nq] tensor-core query rows, the flagged ones gathered in front
  int32_t* qmap;        // [nq] compact row -> query
  int32_t* n_flagged;   // [1]
  uint64_t* vpart_keys; // [kVerifyParts][nq][kk]
};

// Label parts of the compact verify pass (its query rows are few: the parts
// spread them over the SM pairs).
constexpr int kVerifyParts = 64;

// bf16 candidates kept per query before the fp32 re-rank: k' = max(1.5k, k+16),
// a multiple of 8 (bf16 top-k' contains the fp32 top-k; see tests + DESIGN.md).
int rerank_candidates(int k) {
  int kc = std::max((3 * k + 1) / 2, k + 16);
  kc = (kc + 7) / 8 * 8;
  return std::min(kc, 2048);
}

// e4m3 candidate scores are coarser (3 mantissa bits: ~5% of the score spread
// as noise for random data, against ~0.3% for bf16): k' = max(2k, k+32).
int rerank_candidates_f8(int k) {
  int kc = std::max(2 * k, k + 32);
  kc = (kc + 7) / 8 * 8;
  return std::min(kc, 2048);
}

int simt_parts(int64_t nq, int64_t L) {
  const int64_t qtiles = (nq + kBM - 1) / kBM;
  int64_t parts = std::max<int64_t>(1, (2LL * num_sms() + qtiles - 1) / qtiles);
  parts = std::min<int64_t>(parts, std::max<int64_t>(1, (L + kBN - 1) / kBN));
  return static_cast<int>(parts);
}

// Two-pass refresh plan. The exact running top-k spends most of its time in
// data-dependent compaction bursts that stall the tensor pipe (the MMA waits
// for the slowest of four epilogue warps). The two-pass plan removes them:
//  1. sample: every kSampleStride-th label tile (~1/16 of the flops) writes
//     its 64-label group maxima; the j-th largest of them, t_q, is a score
//     at least j sampled labels reach, so about j*16 labels overall; j is
//     chosen so that P(fewer than k keys >= t_q) is ~5 sigma small for
//     i.i.d. scores;
//  2. threshold: the full fused GEMM appends every key >= t_q (FIXED mode:
//     a compare per score, no compaction);
//  3. select: exact top-k of each query's candidates, or a flag when fewer
//     than k non-positive candidates exist (or a list overflowed);
//  4. verify: the exact running top-k only for the query tiles holding a
//     flagged query (CTAs of other tiles exit at once).
// The result equals the running top-k for every query, whatever the data.
struct TwoPass {
  bool on = false;
  int64_t stride = 16;
  int j = 0;            // sample depth
  int n_groups = 0;     // 64-label groups in the sample
  int cand_cap = 0;     // per (query, part) candidate capacity
  int sel_max = 0;      // per-query select capacity (power of two)
};

// Tile stride of the sample pass (ASTRA_SAMPLE_STRIDE overrides; measurement aid).
// Auto (default): 16, doubled up to 64 while the sample still covers >= 300
// label tiles (1200 groups): the sample pass costs 1/stride of the threshold
// pass, and the C5 shard's 58.6K tiles need far fewer than 1/16 of them for the
// same 5-sigma threshold (a coarser stride means more candidates per query,
// j * stride, which the select absorbs). C4 (5.1K tiles) stays at 16.
int64_t sample_stride(int64_t n_tiles) {
  static const int64_t v = [] {
    const char* e = getenv("ASTRA_SAMPLE_STRIDE");
    const int64_t x = e ? atoll(e) : 0;
    return x >= 2 && x <= 256 ? x : 0;
  }();
  if (v) return v;
  int64_t st = 16;
  while (st < 64 && n_tiles / (2 * st) >= 300) st *= 2;
  return st;
}
// per-query select capacity (candidates over all parts): 8192 keeps the
// two-pass plan on for k' up to 512 at 9 label parts (the C5 shard's
// top-(k_h + n_c) = 328 -> k' = 496); the select then stages 32 KB of score
// halves + 8 KB of keys per warp (160 KB per 4-warp CTA)
constexpr int kSelMax = 8192;

TwoPass plan_two_pass(int64_t nq, int64_t L, int kk, int n_parts) {
  TwoPass t;
  const int force = [] {
    const char* e = getenv("ASTRA_REFRESH_TWO_PASS");  // 0 = never, 1 = whenever feasible
    return e ? atoi(e) : -1;
  }();
  const int64_t n_tiles = (L + kTcTileLabels - 1) / kTcTileLabels;
  if (force == 0 || kk > 512) return t;
  const int64_t kSampleStride = sample_stride(n_tiles);
  if (n_tiles < kSampleStride * (force == 1 ? 1 : 32)) return t;  // small label sets: running top-k
  const double z = 5.0, m = static_cast<double>(kk) / kSampleStride;
  int j = static_cast<int>(std::ceil(std::pow(z / 2 + std::sqrt(z * z / 4 + m), 2.0)));
  const int64_t n_lt_s = (n_tiles + kSampleStride - 1) / kSampleStride;
  j = static_cast<int>(std::min<int64_t>(j, n_lt_s * 4 / 2));  // at most half the sample's 64-label groups
  if (j < 1) return t;
  const double mean_per_part = static_cast<double>(j) * kSampleStride / n_parts;
  int cap = static_cast<int>(3.0 * mean_per_part + 64.0);
  cap = (cap + 31) / 32 * 32;
  if (static_cast<int64_t>(cap) * n_parts > kSelMax) {
    if (force != 1) return t;  // many parts (small batches): running top-k
    cap = std::max(32, kSelMax / n_parts / 32 * 32);
  }
  t.on = true;
  t.stride = kSampleStride;
  t.j = j;
  t.n_groups = static_cast<int>(n_lt_s * 4);
  t.cand_cap = cap;
  // the select stages at most sel_max candidates per query: the sum of the part
  // capacities, but no more than 3x the expected total (+128) — many small
  // parts (the SM-filling layouts) would otherwise size it to the worst case
  // of every part full at once and cut the select's occupancy (a query with
  // more candidates is flagged and verified exactly)
  const int64_t total_cap = std::min<int64_t>(static_cast<int64_t>(cap) * n_parts,
                                              static_cast<int64_t>(3.0 * j * kSampleStride) + 128);
  int sm = 1;
  while (sm < total_cap) sm <<= 1;
  t.sel_max = std::min(sm, kSelMax);
  return t;
}

size_t carve_refresh(void* base, size_t cap_bytes, int64_t nq, int64_t L, int d, int k, int mode, RefreshWs* w,
                     int* n_parts_out, int* kk_out, TwoPass* tp) {
  Carve c(base, cap_bytes);
  const int kk = mode == ASTRA_REFRESH_BF16_RERANK ? rerank_candidates(k)
                 : mode == ASTRA_REFRESH_FP8_RERANK ? rerank_candidates_f8(k)
                                                    : k;
  const int cap = topk_cap(kk);
  int n_parts;
  size_t n_bufs;  // per-lane candidate buffers
  size_t buf_words;
  size_t pk_words;
  *tp = TwoPass();
  if (mode == ASTRA_REFRESH_FP32_EXACT) {
    n_parts = simt_parts(nq, L);
    n_bufs = static_cast<size_t>((nq + 127) / 128) * n_parts * 128;
    buf_words = n_bufs * (cap + kTopkSlack);
    pk_words = static_cast<size_t>(n_parts) * nq * kk;
  } else {
    int n_ctas;
    refresh_tc_layout(nq, (L + kTcTileLabels - 1) / kTcTileLabels, &n_ctas, &n_parts);
    // (per-lane running-top-k buffers for every CTA: the compact verify runs on all SMs)
    buf_words = static_cast<size_t>(std::max(n_ctas, num_sms())) * 128 * (cap + kTopkSlack);
    pk_words = static_cast<size_t>(n_parts) * nq * kk;
    *tp = plan_two_pass(nq, L, kk, n_parts);
  }
  w->gtau = c.take<uint64_t>(static_cast<size_t>(nq));
  w->qb = mode == ASTRA_REFRESH_FP32_EXACT ? nullptr
          : mode == ASTRA_REFRESH_FP8_RERANK ? static_cast<void*>(c.take<uint8_t>(static_cast<size_t>(nq) * d))
                                             : static_cast<void*>(c.take<uint16_t>(static_cast<size_t>(nq) * d));
  w->bufs = c.take<uint64_t>(buf_words);
  w->part_keys = c.take<uint64_t>(pk_words);
  w->merge_bufs = c.take<uint64_t>(static_cast<size_t>(nq) * (cap + kTopkSlack));
  const bool rerank = mode == ASTRA_REFRESH_BF16_RERANK || mode == ASTRA_REFRESH_FP8_RERANK;
  w->rr_cand = rerank ? c.take<uint64_t>(static_cast<size_t>(nq) * kk) : nullptr;
  w->gmax = nullptr;
  w->tau_keys = w->cand = nullptr;
  w->cand_cnt = w->flags = nullptr;
  w->qc = nullptr;
  w->qmap = w->n_flagged = nullptr;
  w->vpart_keys = nullptr;
  if (tp->on) {
    w->gmax = c.take<uint32_t>(static_cast<size_t>(nq) * tp->n_groups);
    w->tau_keys = c.take<uint64_t>(static_cast<size_t>(nq));
    w->cand = c.take<uint64_t>(static_cast<size_t>(n_parts) * nq * tp->cand_cap);
    w->cand_cnt = c.take<int32_t>(static_cast<size_t>(n_parts) * nq);
    w->flags = c.take<int32_t>(static_cast<size_t>(nq));
    w->qc = c.take<uint16_t>(static_cast<size_t>(nq) * d);
    w->qmap = c.take<int32_t>(static_cast<size_t>(nq));
    w->n_flagged = c.take<int32_t>(4);
    w->vpart_keys = c.take<uint64_t>(static_cast<size_t>(kVerifyParts) * nq * kk);
  }
  *n_parts_out = n_parts;
  *kk_out = kk;
  return c.off;
}

// Merge of the compact verify's part lists (rows < *n_active, k <= 512) into
// the original queries' outputs (qmap).
int topk_merge_compact(const uint64_t* part_keys, int64_t nq, int n_parts, int k, uint64_t* out_keys, int32_t* out_ids,
                       float* out_scores, const int32_t* qmap, const int32_t* n_active, cudaStream_t st) {
  if (nq <= 0) return ASTRA_OK;
  if (k > 512) return set_error(ASTRA_ERR_CONFIG, "compact verify merge: k > 512");
  const unsigned grid = static_cast<unsigned>((nq + 7) / 8);
  auto go = [&](auto r_tag) {
    constexpr int R = decltype(r_tag)::value;
    merge_warp_kernel<R><<<grid, 256, 0, st>>>(part_keys, nq, n_parts, k, k, out_keys, out_ids, out_scores, nullptr,
                                               qmap, n_active);
  };
  if (k <= 32) go(std::integral_constant<int, 1>());
  else if (k <= 64) go(std::integral_constant<int, 2>());
  else if (k <= 128) go(std::integral_constant<int, 4>());
  else if (k <= 256) go(std::integral_constant<int, 8>());
  else go(std::integral_constant<int, 16>());
  ASTRA_LAUNCHED("merge_compact");
  return ASTRA_OK;
}

int topk_merge_only(const uint64_t* part_keys, int64_t nq, int n_parts, int k_in, int k_out, uint64_t* out_keys,
                    int32_t* out_ids, float* out_scores, uint64_t* bufs, const int32_t* only, cudaStream_t st) {
  if (nq <= 0) return ASTRA_OK;
  if (k_out <= 512) {
    // part lists are sorted descending (refresh / flush output contract)
    const unsigned grid = static_cast<unsigned>((nq + 7) / 8);
    if (k_out <= 32)
      merge_warp_kernel<1><<<grid, 256, 0, st>>>(part_keys, nq, n_parts, k_in, k_out, out_keys, out_ids, out_scores, only);
    else if (k_out <= 64)
      merge_warp_kernel<2><<<grid, 256, 0, st>>>(part_keys, nq, n_parts, k_in, k_out, out_keys, out_ids, out_scores, only);
    else if (k_out <= 128)
      merge_warp_kernel<4><<<grid, 256, 0, st>>>(part_keys, nq, n_parts, k_in, k_out, out_keys, out_ids, out_scores, only);
    else if (k_out <= 256)
      merge_warp_kernel<8><<<grid, 256, 0, st>>>(part_keys, nq, n_parts, k_in, k_out, out_keys, out_ids, out_scores, only);
    else
      merge_warp_kernel<16><<<grid, 256, 0, st>>>(part_keys, nq, n_parts, k_in, k_out, out_keys, out_ids, out_scores, only);
    ASTRA_LAUNCHED("merge_warp");
    return ASTRA_OK;
  }
  if (only) return set_error(ASTRA_ERR_CONFIG, "merge: k_out > 512 with a query subset is not supported");
  const int cap = topk_cap(k_out);
  merge_kernel<<<static_cast<unsigned>((nq + 127) / 128), 128, 0, st>>>(part_keys, nq, n_parts, k_in, k_out, cap,
                                                                       bufs, out_keys, out_ids, out_scores);
  ASTRA_LAUNCHED("merge");
  return ASTRA_OK;
}

}  // namespace

int f32_to_bf16(const float* src, uint16_t* dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return ASTRA_OK;
  const int grid = static_cast<int>(std::min<int64_t>((n / 4 + 255) / 256 + 1, 16LL * num_sms()));
  f32_to_bf16_kernel<<<grid, 256, 0, st>>>(src, dst, n);
  ASTRA_LAUNCHED("f32_to_bf16");
  return ASTRA_OK;
}

// The label snapshot of the FP8_RERANK refresh: n values (fp32 or bf16,
// n % 4 == 0, 16-byte aligned) -> e4m3 bytes scaled by 448 / max|x| (global,
// computed on the device; no host sync). scratch: 2 device words, [1] = the
// scale used (a uniform scale: rankings unchanged).
int quantize_e4m3(const void* src, int src_bf16, int64_t n, uint8_t* dst, float* scratch, cudaStream_t st) {
  if (n < 0 || (n & 3)) return set_error(ASTRA_ERR_CONFIG, "quantize_e4m3: n must be a multiple of 4");
  if (n == 0) return ASTRA_OK;
  if (!src || !dst || !scratch) return set_error(ASTRA_ERR_CONFIG, "quantize_e4m3: null buffer");
  if ((reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 3))
    return set_error(ASTRA_ERR_CONFIG, "quantize_e4m3: misaligned buffers");
  unsigned* bits = reinterpret_cast<unsigned*>(scratch);
  ASTRA_TRY(check_cuda(cudaMemsetAsync(bits, 0, sizeof(unsigned), st), "memset absmax"));
  const int grid = 8 * num_sms();
  if (src_bf16) {
    absmax_kernel<true><<<grid, 256, 0, st>>>(src, n, bits);
    quant_e4m3_kernel<true><<<grid, 256, 0, st>>>(src, n, bits, scratch + 1, dst);
  } else {
    absmax_kernel<false><<<grid, 256, 0, st>>>(src, n, bits);
    quant_e4m3_kernel<false><<<grid, 256, 0, st>>>(src, n, bits, scratch + 1, dst);
  }
  ASTRA_LAUNCHED("quant_e4m3");
  return ASTRA_OK;
}

size_t refresh_workspace_size(int64_t nq, int64_t L, int d, int k, int mode) {
  RefreshWs w;
  int np, kk;
  TwoPass tp;
  return carve_refresh(nullptr, 0, nq, L, d, k, mode, &w, &np, &kk, &tp);
}

int topk_merge(const uint64_t* part_keys, int64_t nq, int n_parts, int k_in, int k_out, uint64_t* out_keys,
               int32_t* out_ids, float* out_scores, uint64_t* bufs, cudaStream_t st) {
  return topk_merge_only(part_keys, nq, n_parts, k_in, k_out, out_keys, out_ids, out_scores, bufs, nullptr, st);
}

// ASTRA_PROFILE_REFRESH=1: CUDA events between the pipeline stages of each
// refresh call, printed after a sync (diagnostics only; changes timing).
struct StageProf {
  bool on = false;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[12];
  const char* name[12];
  int n = 0;
  explicit StageProf(cudaStream_t s) : st(s) {
    static const bool env = getenv("ASTRA_PROFILE_REFRESH") != nullptr;
    on = env;
    if (on) mark("start");
  }
  void mark(const char* what) {
    if (!on || n >= 12) return;
    cudaEventCreate(&ev[n]);
    cudaEventRecord(ev[n], st);
    name[n++] = what;
  }
  ~StageProf() {
    if (!on) return;
    cudaEventSynchronize(ev[n - 1]);
    fprintf(stderr, "[refresh stages]");
    for (int i = 1; i < n; ++i) {
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      fprintf(stderr, " %s=%.3f", name[i], ms);
    }
    float tot = 0.0f;
    cudaEventElapsedTime(&tot, ev[0], ev[n - 1]);
    fprintf(stderr, " total=%.3f ms\n", tot);
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
  }
};

// Stages of the label-sharded BF16 candidate pass (engine._refresh_sharded):
//  1 = the sample pass only, this shard's top-j sampled group maxima per query;
//  2 = the threshold pass with the caller's (global) per-query thresholds and
//      a local select (counts of non-positive candidates kept, overflow flags,
//      no verify);
//  3 = the verify pass for the caller's (global) flags, into out_keys.
struct ShardStage {
  int stage = 0;
  uint32_t* sample_top = nullptr;
  const uint64_t* tau_ext = nullptr;
  int32_t* counts = nullptr;
  int32_t* flags_out = nullptr;
  const int32_t* flags_in = nullptr;
};

int refresh_impl(const float* qf, const uint16_t* qb_in, int64_t nq, int d, const float* wf, const uint16_t* wb,
                 const uint8_t* w8, int64_t L, int64_t off, const int64_t* pos_indptr, const int32_t* pos_ids, int k,
                 int mode, uint64_t* out_keys, int32_t* out_ids, float* out_scores, void* ws, size_t ws_bytes,
                 cudaStream_t st, const ShardStage& ss);

int refresh_topk(const float* qf, const uint16_t* qb_in, int64_t nq, int d, const float* wf, const uint16_t* wb,
                 const uint8_t* w8, int64_t L, int64_t off, const int64_t* pos_indptr, const int32_t* pos_ids, int k,
                 int mode, uint64_t* out_keys, int32_t* out_ids, float* out_scores, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  return refresh_impl(qf, qb_in, nq, d, wf, wb, w8, L, off, pos_indptr, pos_ids, k, mode, out_keys, out_ids,
                      out_scores, ws, ws_bytes, st, ShardStage());
}

// j of the sharded sample statistics (0: this shape does not run the two-pass plan)
int refresh_plan_j(int64_t nq, int64_t L, int d, int k) {
  RefreshWs w;
  int n_parts, kk;
  TwoPass tp;
  (void)carve_refresh(nullptr, 0, nq, L, d, k, ASTRA_REFRESH_BF16, &w, &n_parts, &kk, &tp);
  return tp.on ? tp.j : 0;
}

int refresh_sharded_stage(int stage, const float* qf, const uint16_t* qb, int64_t nq, int d, const uint16_t* wb,
                          int64_t L, int64_t off, const int64_t* pos_indptr, const int32_t* pos_ids, int k,
                          uint32_t* sample_top, const uint64_t* tau_keys, uint64_t* io_keys, int32_t* counts,
                          int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t st) {
  ShardStage ss;
  ss.stage = stage;
  ss.sample_top = sample_top;
  ss.tau_ext = tau_keys;
  ss.counts = counts;
  if (stage == 2) ss.flags_out = flags;
  if (stage == 3) ss.flags_in = flags;
  if ((stage == 1 && !sample_top) || (stage == 2 && (!tau_keys || !counts || !flags || !io_keys)) ||
      (stage == 3 && (!flags || !io_keys)) || stage < 1 || stage > 3)
    return set_error(ASTRA_ERR_CONFIG, "sharded refresh stage %d: bad arguments", stage);
  return refresh_impl(qf, qb, nq, d, nullptr, wb, nullptr, L, off, pos_indptr, pos_ids, k, ASTRA_REFRESH_BF16,
                      io_keys, nullptr, nullptr, ws, ws_bytes, st, ss);
}

int refresh_impl(const float* qf, const uint16_t* qb_in, int64_t nq, int d, const float* wf, const uint16_t* wb,
                 const uint8_t* w8, int64_t L, int64_t off, const int64_t* pos_indptr, const int32_t* pos_ids, int k,
                 int mode, uint64_t* out_keys, int32_t* out_ids, float* out_scores, void* ws, size_t ws_bytes,
                 cudaStream_t st, const ShardStage& ss) {
  if (k < 1 || k > 2048) return set_error(ASTRA_ERR_CONFIG, "refresh: k=%d outside [1, 2048]", k);
  if (nq < 0 || L < 0 || d <= 0) return set_error(ASTRA_ERR_CONFIG, "refresh: bad shape");
  if (L + off >= (int64_t(1) << 31)) return set_error(ASTRA_ERR_CONFIG, "refresh: label ids exceed int32");
  if (nq == 0) return ASTRA_OK;  // nothing to score (empty tensors may carry NULL pointers)
  if (mode == ASTRA_REFRESH_FP32_EXACT) {
    if (!qf || !wf) return set_error(ASTRA_ERR_CONFIG, "FP32_EXACT needs fp32 queries and labels");
  } else if (mode == ASTRA_REFRESH_BF16 || mode == ASTRA_REFRESH_BF16_RERANK) {
    if (d % 64) return set_error(ASTRA_ERR_CONFIG, "bf16 refresh needs d %% 64 == 0 (d=%d)", d);
    if (!wb) return set_error(ASTRA_ERR_CONFIG, "bf16 refresh needs the bf16 label snapshot");
    if (!qf && !qb_in) return set_error(ASTRA_ERR_CONFIG, "bf16 refresh needs queries");
    if (mode == ASTRA_REFRESH_BF16_RERANK && !qf) return set_error(ASTRA_ERR_CONFIG, "BF16_RERANK needs fp32 queries");
  } else if (mode == ASTRA_REFRESH_FP8_RERANK) {
    if (d % 128) return set_error(ASTRA_ERR_CONFIG, "e4m3 refresh needs d %% 128 == 0 (d=%d)", d);
    if (!w8) return set_error(ASTRA_ERR_CONFIG, "FP8_RERANK needs the e4m3 label snapshot");
    if (!qf) return set_error(ASTRA_ERR_CONFIG, "FP8_RERANK needs fp32 queries");
    if (!wf && !wb) return set_error(ASTRA_ERR_CONFIG, "FP8_RERANK re-ranks on the fp32 or bf16 labels: give one");
    if (rerank_candidates_f8(k) > 512) return set_error(ASTRA_ERR_CONFIG, "FP8_RERANK needs k' = 2k <= 512 (k <= 256)");
  } else {
    return set_error(ASTRA_ERR_CONFIG, "refresh: unknown mode %d", mode);
  }
  RefreshWs w;
  int n_parts, kk;
  TwoPass tp;
  size_t need = carve_refresh(ws, ws_bytes, nq, L, d, k, mode, &w, &n_parts, &kk, &tp);
  if (!ws || ws_bytes < need) return set_error(ASTRA_ERR_CONFIG, "refresh workspace too small (%zu < %zu)", ws_bytes, need);
  if (nq == 0) return ASTRA_OK;
  StageProf prof(st);
  const int cap = topk_cap(kk);
  // where the bf16 / fp32 top-kk lands: the re-rank input, or the caller's outputs
  const bool rerank = mode == ASTRA_REFRESH_BF16_RERANK || mode == ASTRA_REFRESH_FP8_RERANK;
  const bool f8 = mode == ASTRA_REFRESH_FP8_RERANK;
  if (rerank && !w.rr_cand) return set_error(ASTRA_ERR_CONFIG, "refresh: re-rank staging not carved");
  uint64_t* o_keys = rerank ? w.rr_cand : out_keys;
  int32_t* o_ids = rerank ? nullptr : out_ids;
  float* o_scores = rerank ? nullptr : out_scores;
  if (mode == ASTRA_REFRESH_FP32_EXACT) {
    SimtArgs a;
    a.Q = qf;
    a.W = wf;
    a.nq = nq;
    a.L = L;
    a.off = off;
    a.d = d;
    a.k = kk;
    a.cap = cap;
    a.n_parts = n_parts;
    const int64_t tiles = (L + kBN - 1) / kBN;
    a.labels_per_part = ((tiles + n_parts - 1) / n_parts) * kBN;
    a.pos_indptr = pos_indptr;
    a.pos_ids = pos_ids;
    a.bufs = w.bufs;
    a.part_keys = w.part_keys;
    a.gtau = w.gtau;
    ASTRA_TRY(check_cuda(cudaMemsetAsync(w.gtau, 0, sizeof(uint64_t) * nq, st), "memset gtau"));
    dim3 grid(static_cast<unsigned>((nq + kBM - 1) / kBM), static_cast<unsigned>(n_parts));
    cudaFuncSetAttribute(refresh_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSimtSmem);
    refresh_simt_kernel<<<grid, kSimtThreads, kSimtSmem, st>>>(a);
    ASTRA_LAUNCHED("refresh_simt");
    ASTRA_TRY(topk_merge(w.part_keys, nq, n_parts, kk, kk, o_keys, o_ids, o_scores, w.merge_bufs, st));
  } else {
    const void* qb = qb_in;
    if (f8) {
      quant_rows_e4m3_kernel<<<static_cast<unsigned>((nq + 7) / 8), 256, 0, st>>>(qf, nq, d,
                                                                                 static_cast<uint8_t*>(w.qb));
      ASTRA_LAUNCHED("quant_rows_e4m3");
      qb = w.qb;
    } else if (!qb) {
      ASTRA_TRY(f32_to_bf16(qf, static_cast<uint16_t*>(w.qb), nq * d, st));
      qb = w.qb;
    }
    TcLaunch p;
    p.qb = qb;
    p.nq = nq;
    p.d = d;
    p.wb = f8 ? static_cast<const void*>(w8) : static_cast<const void*>(wb);
    p.f8 = f8;
    p.L = L;
    p.off = off;
    p.pos_indptr = pos_indptr;
    p.pos_ids = pos_ids;
    p.bufs = w.bufs;
    p.part_keys = w.part_keys;
    p.gtau = w.gtau;
    if (ss.stage != 0 && !tp.on)
      return set_error(ASTRA_ERR_CONFIG, "sharded refresh stage %d needs the two-pass plan", ss.stage);
    // 4. verify: the exact running top-k for the flagged queries only,
    //    gathered to the front of a compact query buffer (their number stays
    //    on the device): a handful of flagged queries costs one query-tile
    //    pair's sweep spread over kVerifyParts label parts, not the full
    //    tiles they sit in
    auto verify_pass = [&](const int32_t* vflags) -> int {
      // (near zero unless a query was flagged: bench.py reports it per refresh)
      KernelTimer kt("refresh_verify", st);
      compact_flagged_kernel<<<1, 1024, 0, st>>>(vflags, nq, w.qmap, w.n_flagged);
      ASTRA_LAUNCHED("compact_flagged");
      const int64_t row_bytes = f8 ? d : static_cast<int64_t>(d) * 2;
      gather_rows_kernel<<<static_cast<unsigned>(nq), 128, 0, st>>>(static_cast<const unsigned char*>(qb), row_bytes,
                                                                    w.qmap, w.n_flagged,
                                                                    static_cast<unsigned char*>(w.qc));
      ASTRA_LAUNCHED("gather_rows");
      TcLaunch v = p;
      v.qb = w.qc;
      v.k = kk;
      v.cap = cap;
      v.part_keys = w.vpart_keys;
      v.qmap = w.qmap;
      v.n_active = w.n_flagged;
      v.n_parts_fixed = kVerifyParts;
      ASTRA_TRY(launch_refresh_tc(v, st));
      const int vparts = static_cast<int>(std::min<int64_t>(kVerifyParts, (L + kTcTileLabels - 1) / kTcTileLabels));
      return topk_merge_compact(w.vpart_keys, nq, vparts, kk, o_keys, o_ids, o_scores, w.qmap, w.n_flagged, st);
    };
    if (tp.on && ss.stage == 3) return verify_pass(ss.flags_in);  // (the sharded verify stage: flags given)
    if (tp.on) {
      // 1. sample pass: group maxima of every stride-th label tile, threshold
      //    (sharded stage 2: the threshold comes from the caller)
      if (ss.stage != 2) {
        TcLaunch s = p;
        s.tile_stride = tp.stride;
        s.gmax = w.gmax;
        prof.mark("to_bf16");
        ASTRA_TRY(launch_refresh_tc(s, st));
        prof.mark("sample");
        if (ss.stage == 1) {  // the shard's top-j sampled group maxima per query, for the owners
          sample_top_kernel<<<static_cast<unsigned>((nq + 7) / 8), 256, 0, st>>>(w.gmax, nq, tp.n_groups, tp.j,
                                                                                 ss.sample_top);
          ASTRA_LAUNCHED("sample_top");
          return ASTRA_OK;
        }
        tau_select_kernel<<<static_cast<unsigned>((nq + 7) / 8), 256, 0, st>>>(w.gmax, nq, tp.n_groups, tp.j,
                                                                               w.tau_keys);
        ASTRA_LAUNCHED("tau_select");
      }
      // 2. threshold pass over every label
      TcLaunch f = p;
      f.tau_in = ss.stage == 2 ? ss.tau_ext : w.tau_keys;
      f.tau_stride = 1;
      f.cand = w.cand;
      f.cand_cnt = w.cand_cnt;
      f.cand_cap = tp.cand_cap;
      prof.mark("tau_select");
      {
        KernelTimer kt("refresh_gemm", st);
        ASTRA_TRY(launch_refresh_tc(f, st));
      }
      prof.mark("threshold");
      // 3. select
      const int rcap = sel_rcap(kk);
      const size_t smem = (sizeof(uint64_t) * rcap + sizeof(uint32_t) * tp.sel_max) * kSelWarps;
      cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      select_kernel<<<static_cast<unsigned>((nq + kSelWarps - 1) / kSelWarps), kSelWarps * 32, smem, st>>>(
          w.cand, w.cand_cnt, n_parts, tp.cand_cap, nq, pos_indptr, pos_ids, kk, tp.sel_max, rcap, o_keys, o_ids,
          o_scores, ss.stage == 2 ? ss.flags_out : w.flags, ss.stage == 2 ? ss.counts : nullptr);
      ASTRA_LAUNCHED("select");
      if (ss.stage == 2) return ASTRA_OK;  // (the owners decide which queries to verify)
      prof.mark("select");
      ASTRA_TRY(verify_pass(w.flags));
      prof.mark("verify");
    } else {
      p.k = kk;
      p.cap = cap;
      {
        KernelTimer kt("refresh_gemm", st);
        ASTRA_TRY(launch_refresh_tc(p, st));
      }
      ASTRA_TRY(topk_merge(w.part_keys, nq, n_parts, kk, kk, o_keys, o_ids, o_scores, w.merge_bufs, st));
    }
  }
  static const bool legacy_rr = getenv("ASTRA_RERANK_LEGACY") != nullptr;
  // the re-rank scores the fp32 snapshot, or the bf16 one when no fp32 copy is given (bf16 W)
  const bool rr_bf16 = wf == nullptr;
  const void* wl = rr_bf16 ? static_cast<const void*>(wb) : static_cast<const void*>(wf);
  if (rerank && (rr_bf16 || (!legacy_rr && kk <= 512 && d % 64 == 0 && (reinterpret_cast<uintptr_t>(wf) & 15) == 0))) {
    if (kk > 512) return set_error(ASTRA_ERR_CONFIG, "BF16_RERANK from bf16 labels needs k' <= 512 (k <= 341)");
    auto go = [&](auto r_tag) {
      constexpr int R = decltype(r_tag)::value;
      return rr_bf16 ? launch_rerank_tma<R, true>(qf, wl, d, off, w.rr_cand, nq, kk, k, out_keys, out_ids, out_scores, st)
                     : launch_rerank_tma<R, false>(qf, wl, d, off, w.rr_cand, nq, kk, k, out_keys, out_ids, out_scores,
                                                   st);
    };
    int rc;
    if (kk <= 32)
      rc = go(std::integral_constant<int, 1>());
    else if (kk <= 64)
      rc = go(std::integral_constant<int, 2>());
    else if (kk <= 128)
      rc = go(std::integral_constant<int, 4>());
    else if (kk <= 256)
      rc = go(std::integral_constant<int, 8>());
    else
      rc = go(std::integral_constant<int, 16>());
    prof.mark("rerank");
    return rc;
  }
  if (rerank) {
    int Pn = 1;
    while (Pn < kk) Pn <<= 1;
    size_t smem = align_up(sizeof(float) * (d + kRrWarps * 32 * kRrPitch), 16) + sizeof(uint64_t) * Pn;
    if (smem > 48 * 1024) cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rerank_kernel<<<static_cast<unsigned>(nq), kRrWarps * 32, smem, st>>>(qf, wf, d, off, w.rr_cand, kk, k, out_keys,
                                                                           out_ids, out_scores);
    ASTRA_LAUNCHED("rerank");
  }
  return ASTRA_OK;
}

// Queries of the last two-pass refresh that used this workspace whose
// candidate set could not prove exactness (the running-top-k verify re-did
// them): copies the flags back and counts them (synchronises the stream).
// -1 when the plan for this shape is not the two-pass one.
int refresh_flagged(const void* ws, size_t ws_bytes, int64_t nq, int64_t L, int d, int k, int mode,
                    int64_t* out_count, cudaStream_t st) {
  if (!out_count) return set_error(ASTRA_ERR_CONFIG, "refresh_flagged: null output");
  *out_count = -1;
  if (mode == ASTRA_REFRESH_FP32_EXACT || nq <= 0) return ASTRA_OK;
  RefreshWs w;
  int n_parts, kk;
  TwoPass tp;
  size_t need = carve_refresh(const_cast<void*>(ws), ws_bytes, nq, L, d, k, mode, &w, &n_parts, &kk, &tp);
  if (!ws || ws_bytes < need) return set_error(ASTRA_ERR_CONFIG, "refresh_flagged: workspace too small");
  if (!tp.on) return ASTRA_OK;
  std::vector<int32_t> h(static_cast<size_t>(nq));
  ASTRA_TRY(check_cuda(cudaMemcpyAsync(h.data(), w.flags, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st), "flags d2h"));
  ASTRA_TRY(check_cuda(cudaStreamSynchronize(st), "flags sync"));
  int64_t c = 0;
  for (int32_t f : h) c += f != 0;
  *out_count = c;
  return ASTRA_OK;
}

}  // namespace astra
