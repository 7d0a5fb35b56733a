// sampler.cu — Philox4x32-10 negative-mixture sampler.
//
// Replaces the PCG64 slate assembly of the reference,
// _assemble_batch_slates (trainer.py:262-318) / assemble_slate
// (sampler.py:146-186), with a counter-based stream so every (row, slot)
// draw is independent of batch composition and of the thread that makes it.
// One CTA per batch row; the row's hard (+candidate) set is sorted once in
// shared memory and every uniform draw maps rank -> id by binary search
// (trainer.py:300-306). Draw-for-draw equal to oracle_sample_slates.
#include <limits.h>

#include "common.cuh"
#include "ptx.cuh"

namespace astra {
namespace {

constexpr uint32_t TAG_POSKEY = 1, TAG_PAD = 2, TAG_IMP = 3, TAG_RAND = 4;
constexpr int kThreads = 128;
constexpr int kMaxSet = 4096;  // |hard| + |cand| per row
constexpr int kSmemPos = 256;  // a row's positives staged in shared memory up to this many

struct SamplerArgs {
  uint32_t k0, k1, epoch, step;
  const int64_t* rows;
  const int64_t* pos_indptr;
  const int32_t* pos_ids;
  const int32_t* hard;
  int hard_stride, k_h;
  const int32_t* cand;
  const float* cand_q;
  int cand_stride, n_c, k_i;
  int64_t L;
  int k_p, k_r, S, m, P;
  int32_t* ids;
  int8_t* y;
  int8_t* origin;
  float* weights;
};

__device__ __forceinline__ U4 draw(const SamplerArgs& a, uint32_t row, uint32_t c0, uint32_t tag) {
  return philox4x32_10(c0, row, a.epoch, (tag << 24) | (a.step & 0xFFFFFFu), a.k0, a.k1);
}

__global__ void __launch_bounds__(kThreads) sample_slates_kernel(SamplerArgs a) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem[];
  double* cdf = reinterpret_cast<double*>(smem);                     // n_c
  int32_t* C = reinterpret_cast<int32_t*>(smem + sizeof(double) * a.n_c);  // P, sorted hard (+cand)
  __shared__ double s_total;
  __shared__ int32_t s_pos[kSmemPos];

  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  const uint32_t row = static_cast<uint32_t>(a.rows[b]);
  const int32_t* pos_g = a.pos_ids + a.pos_indptr[b];
  const int64_t npos = a.pos_indptr[b + 1] - a.pos_indptr[b];
  // the row's sorted positives, searched by every pad / uniform / importance
  // draw: from shared memory unless the row has more than kSmemPos of them
  if (npos <= kSmemPos)
    for (int j = tid; j < npos; j += kThreads) s_pos[j] = pos_g[j];
  const int32_t* pos = npos <= kSmemPos ? s_pos : pos_g;
  const bool use_cand = a.k_i > 0 && a.n_c > 0;
  const size_t base = static_cast<size_t>(b) * a.S;

  // -- the excluded set C, sorted ascending (bitonic in shared memory)
  for (int j = tid; j < a.P; j += kThreads) {
    int32_t v = INT_MAX;
    if (j < a.k_h)
      v = a.hard[static_cast<size_t>(b) * a.hard_stride + j];
    else if (use_cand && j < a.m)
      v = a.cand[static_cast<size_t>(b) * a.cand_stride + (j - a.k_h)];
    C[j] = v;
  }
  __syncthreads();
  for (int size = 2; size <= a.P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < a.P; i += kThreads) {
        int j = i ^ stride;
        if (j > i) {
          bool up = (i & size) == 0;
          int32_t x = C[i], z = C[j];
          if ((x > z) == up) {
            C[i] = z;
            C[j] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  // -- importance CDF (sequential fp64, identical to the oracle)
  if (tid == 0) {
    double tot = 0.0;
    if (use_cand)
      for (int c = 0; c < a.n_c; ++c) {
        tot += static_cast<double>(a.cand_q[static_cast<size_t>(b) * a.cand_stride + c]);
        cdf[c] = tot;
      }
    s_total = tot;
  }
  // -- positive subset: the min(npos, k_p) smallest (philox key, index) pairs
  //    in increasing order = a uniformly random ordered subset (trainer.py:273-281)
  if (tid < 32) {
    const int take = static_cast<int>(npos < a.k_p ? npos : a.k_p);
    auto poskey = [&](int64_t p) {
      return (static_cast<uint64_t>(draw(a, row, static_cast<uint32_t>(p), TAG_POSKEY).x) << 32) |
             static_cast<uint32_t>(p);
    };
    // rows with <= 64 positives: every key drawn once, held in registers
    const bool cached = npos <= 64;
    uint64_t k0 = ~0ull, k1 = ~0ull;
    if (cached && take > 0) {
      if (tid < npos) k0 = poskey(tid);
      if (tid + 32 < npos) k1 = poskey(tid + 32);
    }
    uint64_t prev = 0;
    bool first = true;
    for (int r = 0; r < take; ++r) {
      uint64_t best = ~0ull;
      if (cached) {
        if ((first || k0 > prev) && k0 < best) best = k0;
        if ((first || k1 > prev) && k1 < best) best = k1;
      } else {
        for (int64_t p = tid; p < npos; p += 32) {
          const uint64_t kp = poskey(p);
          if ((first || kp > prev) && kp < best) best = kp;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        uint64_t other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
      }
      if (tid == 0) {
        a.ids[base + r] = pos[static_cast<uint32_t>(best)];
        a.y[base + r] = 1;
        a.origin[base + r] = ASTRA_ORIGIN_POS;
        a.weights[base + r] = 1.0f;
      }
      prev = best;
      first = false;
    }
  }
  // Without importance draws nothing below depends on warp 0's work (the
  // subset above writes slots [0, min(npos, k_p)), skipped below): warps 1..
  // take every other slot and run concurrently with it, no barrier.
  const bool split = !use_cand;
  if (!split) __syncthreads();  // the CDF (thread 0)
  if (split && tid < 32) return;

  const double tot = split ? 0.0 : s_total;
  const float w_rand = a.k_r > 0 ? static_cast<float>(static_cast<double>(a.L - a.m) / a.k_r) : 0.0f;
  const int h0 = a.k_p, i0 = a.k_p + a.k_h, r0 = a.k_p + a.k_h + a.k_i;
  const int j0 = split ? tid - 32 : tid, jstep = split ? kThreads - 32 : kThreads;
  for (int j = j0; j < a.S; j += jstep) {
    int32_t id;
    int8_t yy, oo;
    float ww;
    if (j < a.k_p) {
      if (j < npos) continue;  // written by warp 0
      // pad: uniform over [0, L) rejecting the row's positives (trainer.py:283-290)
      uint32_t att = 0;
      int64_t v;
      do {
        v = static_cast<int64_t>(bounded_u64(draw(a, row, static_cast<uint32_t>(j) | (att << 20), TAG_PAD),
                                             static_cast<uint64_t>(a.L)));
        ++att;
      } while (sorted_contains(pos, npos, v));
      id = static_cast<int32_t>(v);
      yy = 0;
      oo = ASTRA_ORIGIN_PAD;
      ww = 1.0f;
    } else if (j < i0) {
      id = a.hard[static_cast<size_t>(b) * a.hard_stride + (j - h0)];  // trainer.py:295-298
      yy = 0;
      oo = ASTRA_ORIGIN_HARD;
      ww = 1.0f;
    } else if (j < r0) {
      int c = 0;
      double q = 1.0;
      if (use_cand) {
        U4 r = draw(a, row, static_cast<uint32_t>(j), TAG_IMP);
        uint64_t x = static_cast<uint64_t>(r.x) | (static_cast<uint64_t>(r.y) << 32);
        double target = static_cast<double>(x >> 11) * 0x1.0p-53 * tot;
        int lo = 0, hi = a.n_c - 1;
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (cdf[mid] > target)
            hi = mid;
          else
            lo = mid + 1;
        }
        c = lo;
        q = static_cast<double>(a.cand_q[static_cast<size_t>(b) * a.cand_stride + c]);
      }
      id = use_cand ? a.cand[static_cast<size_t>(b) * a.cand_stride + c] : 0;
      yy = static_cast<int8_t>(sorted_contains(pos, npos, id));
      oo = ASTRA_ORIGIN_IMP;
      ww = use_cand ? static_cast<float>(tot / (static_cast<double>(a.k_i) * q)) : 0.0f;
    } else {
      // uniform over [L] \ C: v + #{t : C[t] - t <= v}  (trainer.py:300-306)
      int64_t v = static_cast<int64_t>(
          bounded_u64(draw(a, row, static_cast<uint32_t>(j), TAG_RAND), static_cast<uint64_t>(a.L - a.m)));
      int lo = 0, hi = a.m;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (static_cast<int64_t>(C[mid]) - mid <= v)
          lo = mid + 1;
        else
          hi = mid;
      }
      id = static_cast<int32_t>(v + lo);
      yy = static_cast<int8_t>(sorted_contains(pos, npos, id));  // trainer.py:309
      oo = ASTRA_ORIGIN_RAND;
      ww = w_rand;  // trainer.py:315-317
    }
    a.ids[base + j] = id;
    a.y[base + j] = yy;
    a.origin[base + j] = oo;
    a.weights[base + j] = ww;
  }
}

}  // namespace

int sample_slates(uint64_t seed, uint32_t epoch, uint32_t step, const int64_t* rows, int B,
                  const int64_t* pos_indptr, const int32_t* pos_ids, const int32_t* hard, int hard_stride,
                  int k_h, const int32_t* cand, const float* cand_q, int cand_stride, int n_c, int k_i,
                  int64_t n_labels, int k_p, int k_r, int32_t* ids, int8_t* y, int8_t* origin, float* weights,
                  cudaStream_t stream) {
  if (B < 0 || k_p < 0 || k_h < 0 || k_i < 0 || k_r < 0 || n_c < 0)
    return set_error(ASTRA_ERR_CONFIG, "sampler: negative count");
  if (k_h > 0 && (!hard || hard_stride < k_h)) return set_error(ASTRA_ERR_CONFIG, "sampler: hard rows missing");
  const bool use_cand = k_i > 0 && n_c > 0;
  if (k_i > 0 && (!cand || !cand_q || cand_stride < n_c))
    return set_error(ASTRA_ERR_CONFIG, "sampler: importance candidates missing");
  const int m = k_h + (use_cand ? n_c : 0);
  if (m > kMaxSet) return set_error(ASTRA_ERR_CONFIG, "sampler: |hard|+|cand| = %d exceeds %d", m, kMaxSet);
  if (static_cast<int64_t>(m) >= n_labels)
    return set_error(ASTRA_ERR_CONFIG, "hard set covers the whole label space");  // sampler.py:120-121
  if (B == 0) return ASTRA_OK;
  SamplerArgs a;
  a.k0 = static_cast<uint32_t>(seed);
  a.k1 = static_cast<uint32_t>(seed >> 32);
  a.epoch = epoch;
  a.step = step;
  a.rows = rows;
  a.pos_indptr = pos_indptr;
  a.pos_ids = pos_ids;
  a.hard = hard;
  a.hard_stride = hard_stride;
  a.k_h = k_h;
  a.cand = cand;
  a.cand_q = cand_q;
  a.cand_stride = cand_stride;
  a.n_c = use_cand ? n_c : 0;
  a.k_i = k_i;
  a.L = n_labels;
  a.k_p = k_p;
  a.k_r = k_r;
  a.S = k_p + k_h + k_i + k_r;
  a.m = m;
  int P = 1;
  while (P < m) P <<= 1;
  a.P = m > 0 ? P : 0;
  a.ids = ids;
  a.y = y;
  a.origin = origin;
  a.weights = weights;
  size_t smem = sizeof(double) * a.n_c + sizeof(int32_t) * a.P;
  launch_pdl(sample_slates_kernel, B, kThreads, smem, stream, a);
  ASTRA_LAUNCHED("sample_slates_kernel");
  return ASTRA_OK;
}

// ------------------------------------------------------------- importance cache
// The stale refresh of top-(k_h + n_c) per row (ids + fp32 scores, descending)
// becomes the row's negative-mixture cache: the first k_h
// ids are the hard set H, the next n_c the importance candidates C with
// stored probability weights q_c = sigmoid(stale score_c) (the sampler
// normalises them per row). Missing entries (id < 0: fewer labels than asked)
// get q = 0 and are never drawn.
__global__ void importance_split_kernel(const int32_t* ids, const float* scores, int64_t nq, int k_tot, int k_h,
                                        int32_t* hard, int32_t* cand, float* cand_q) {
  const int n_c = k_tot - k_h;
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nq * k_tot) return;
  const int64_t r = i / k_tot;
  const int j = static_cast<int>(i - r * k_tot);
  const int32_t id = ids[i];
  if (j < k_h) {
    hard[r * k_h + j] = id;
  } else {
    const int c = j - k_h;
    cand[r * n_c + c] = id;
    cand_q[r * n_c + c] = id >= 0 ? 1.0f / (1.0f + expf(-scores[i])) : 0.0f;
  }
}

int importance_split(const int32_t* ids, const float* scores, int64_t nq, int k_tot, int k_h, int32_t* hard,
                     int32_t* cand, float* cand_q, cudaStream_t st) {
  if (nq < 0 || k_h < 0 || k_tot < k_h) return set_error(ASTRA_ERR_CONFIG, "importance_split: bad sizes");
  if (nq == 0 || k_tot == 0) return ASTRA_OK;
  if (!ids || !scores || (k_h && !hard) || (k_tot > k_h && (!cand || !cand_q)))
    return set_error(ASTRA_ERR_CONFIG, "importance_split: null buffer");
  const int64_t n = nq * k_tot;
  importance_split_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(ids, scores, nq, k_tot, k_h, hard,
                                                                                   cand, cand_q);
  ASTRA_LAUNCHED("importance_split");
  return ASTRA_OK;
}

}  // namespace astra
