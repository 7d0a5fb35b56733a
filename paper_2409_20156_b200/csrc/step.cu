// step.cu — sampled BCE forward/backward fused with the sparse row update.
//
// Replaces the classifier half of _batch_forward_backward
// (trainer.py:366-394) and apply_classifier_updates_arrays
// (classifiers.py:75-82). HBM-bound. Per minibatch:
//
//   count/scan/scatter  counting sort of the B*S slots by local label
//                     (replaces the dense L x d A^T@emb, trainer.py:390-393);
//                     count also accumulates the finiteness bounds and
//                     scan_top decides the schedule on the device.
//   step_single_tma   (default for SGD, d % 128 == 0) ONE label-major pass:
//                     per unique label, the old row is bulk-copied once; every
//                     occurrence's score, loss term, factor, grad_emb[b] +=
//                     f * W_old (vector reductions) and g += f * emb_b; then
//                     the SGD/Adam row update and store: each touched row read
//                     and written once.
//   two-kernel schedule (deterministic / Adam / when the bound proof fails):
//     slot_forward    (CTA per batch row) gather W[ids[b,s]], dot, BCE loss
//                     terms (fp64), factors c*(sigma-y) (trainer.py:369-380),
//                     grad_emb[b] in a fixed order (trainer.py:382-384);
//     finalize        fixed-order fp64 loss sum + overflow bound;
//     label_update    (per unique label) sum f*emb in ascending b*S+s order
//                     with separate mul/add roundings — scipy's csc_matvecs
//                     order — then the SGD/Adam row update.
// W is written only if every touched gradient and grad_emb is finite: the
// reference raises NumericalError before writing (classifiers.py:79-80,
// encoder.py:145-146): the single pass proves it from bounds up front; the
// two-kernel schedule checks first (label_check) when its bound trips.
#include <atomic>
#include <limits.h>
#include <math.h>

#include <cmath>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace astra {
namespace {

constexpr int kFwdThreads = 256;
constexpr int kFwdWarps = kFwdThreads / 32;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr int kUpdThreads = 256;
constexpr double kBoundSafe = 1e37;
constexpr double kSingleSafe = 1e30;  // single-pass schedule: bound on every |gradient| entry

struct FwdArgs {
  const float* emb;
  const float* keep;
  const int32_t* ids;
  const int8_t* y;
  const int8_t* origin;
  int64_t origin_stride;
  const float* weights;
  int64_t weights_stride;
  const float* factors_in;
  int B, S, d;
  const void* W;
  int64_t Lloc, off;
  float* grad_emb;
  float* factors;
  double* loss_rows;
  double* bound_rows;
  int32_t* status;
  const int32_t* skip = nullptr;  // != null and *skip: the single-pass schedule ran (kernel returns)
};

__device__ __forceinline__ float expit_f32(float x) {
  // scipy.special.expit on float32: 1 / (1 + exp(-x)) in single precision
  // (the correctly rounded reciprocal = the correctly rounded 1/y division, bit
  // for bit, without the division's numerator scaling and slow-path branch)
  return __frcp_rn(__fadd_rn(1.0f, expf(-x)));
}

__device__ __forceinline__ double softplus64(double x) {
  // log(1 + e^x) = logaddexp(0, x) (loss.py:36-43)
  return fmax(x, 0.0) + log1p(exp(-fabs(x)));
}

// d(loss)/d(score) and the fp64 loss term of one slot (trainer.py:369-380).
__device__ __forceinline__ float slot_factor(const FwdArgs& a, int b, int s, float sc, double* loss_term) {
  const int8_t o = a.origin[b * a.origin_stride + s];
  const float yf = static_cast<float>(a.y[static_cast<size_t>(b) * a.S + s]);
  const float w = a.weights[b * a.weights_stride + s];
  const bool pos_slot = o == ASTRA_ORIGIN_POS;
  const float pos_term = pos_slot ? yf : 0.0f;
  const float neg_alive = pos_slot ? 0.0f : __fsub_rn(1.0f, yf);
  const float sig = expit_f32(sc);
  const float wn = __fmul_rn(w, neg_alive);
  const double spn = softplus64(-static_cast<double>(sc));
  *loss_term = static_cast<double>(pos_term) * spn + static_cast<double>(wn) * (spn + static_cast<double>(sc));
  return __fadd_rn(__fmul_rn(pos_term, __fsub_rn(sig, 1.0f)), __fmul_rn(wn, sig));
}

// The slot's (origin, y, weight), loaded ahead of its W row so that these
// L2 loads overlap the row's arrival instead of following it.
struct SlotMeta {
  int8_t o;
  float yf, w;
};

__device__ __forceinline__ SlotMeta slot_meta(const FwdArgs& a, int b, int s) {
  SlotMeta m;
  m.o = a.origin[b * a.origin_stride + s];
  m.yf = static_cast<float>(a.y[static_cast<size_t>(b) * a.S + s]);
  m.w = a.weights[b * a.weights_stride + s];
  return m;
}

// The factor (needed at once by every lane) from prefetched metadata; the fp64
// loss term is evaluated later, lane-parallel for 32 slots at a time.
__device__ __forceinline__ float slot_factor_meta(const SlotMeta& m, float sc, float* pos_term_out, float* wn_out) {
  const bool pos_slot = m.o == ASTRA_ORIGIN_POS;
  const float pos_term = pos_slot ? m.yf : 0.0f;
  const float neg_alive = pos_slot ? 0.0f : __fsub_rn(1.0f, m.yf);
  const float sig = expit_f32(sc);
  const float wn = __fmul_rn(m.w, neg_alive);
  *pos_term_out = pos_term;
  *wn_out = wn;
  return __fadd_rn(__fmul_rn(pos_term, __fsub_rn(sig, 1.0f)), __fmul_rn(wn, sig));
}

__device__ __forceinline__ double slot_loss(float sc, float pos_term, float wn) {
  const double spn = softplus64(-static_cast<double>(sc));
  return static_cast<double>(pos_term) * spn + static_cast<double>(wn) * (spn + static_cast<double>(sc));
}

// Hot labels (more than kHotOcc occurrences in the minibatch, e.g. the
// popular rows of a clustered, trained W that many rows' hard lists share):
// the single pass would walk their occurrences serially on one warp and rank-
// sort them in O(n^2); they go to hot_label_kernel instead (block per label:
// occurrences scored in parallel, then the ordered gradient sum), up to
// kHotMax occurrences (its shared-memory sort).
constexpr uint32_t kHotOcc = 32, kHotMax = 8192;
__host__ __device__ __forceinline__ bool is_hot(uint32_t n) { return n > kHotOcc && n <= kHotMax; }

// Ring slots are released (mbarrier arrive, then refilled by a TMA bulk copy:
// the async proxy) right after a warp's shared-memory loads of the slot. An
// LDS still in flight at the arrive could read the next fill: each lane first
// waits for its loaded registers (an empty asm that consumes them), then the
// warp syncs and lane 0 arrives. (compute-sanitizer racecheck flagged these
// read/bulk-write pairs; a rare wrong Adam update fit the same window.)
template <int N>
__device__ __forceinline__ void regs_landed(const float4 (&r)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" ::"f"(r[i].x), "f"(r[i].y), "f"(r[i].z), "f"(r[i].w) : "memory");
  fence_proxy_async_smem();
}

template <bool BF16>
__device__ __forceinline__ float4 load_w4(const void* W, size_t elem) {
  if constexpr (BF16) {
    uint2 u = __ldg(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(W) + elem));
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                       __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
  } else {
    return __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(W) + elem));
  }
}

// Shared tail of both forward kernels: reduce the per-warp grad_emb / loss /
// |f| partials in warp order (deterministic) and write row b.
__device__ void forward_tail(const FwdArgs& a, int b, float* red, double lsum, double fabs_sum, float emax) {
  __shared__ double s_loss[kFwdWarps], s_fabs[kFwdWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  lsum = warp_sum(lsum);
  fabs_sum = warp_sum(fabs_sum);
  if (lane == 0) {
    s_loss[warp] = lsum;
    s_fabs[warp] = fabs_sum;
  }
  __syncthreads();
  bool bad = false;
  for (int k = threadIdx.x; k < a.d; k += kFwdThreads) {
    float g = 0.0f;
#pragma unroll
    for (int w = 0; w < kFwdWarps; ++w) g += red[w * a.d + k];
    if (a.keep) g = __fmul_rn(g, a.keep[static_cast<size_t>(b) * a.d + k]);
    a.grad_emb[static_cast<size_t>(b) * a.d + k] = g;
    bad |= !isfinite(g);
  }
  if (bad) a.status[ASTRA_STATUS_NONFINITE_GRAD_EMB] = 1;
  if (threadIdx.x == 0) {
    double l = 0.0, fa = 0.0;
    for (int w = 0; w < kFwdWarps; ++w) {
      l += s_loss[w];
      fa += s_fabs[w];
    }
    a.loss_rows[b] = l;
    a.bound_rows[b] = fa * static_cast<double>(emax);
  }
}

// TMA-fed forward (the default for d % 128 == 0): CTA per batch row; one
// producer lane streams the row's owned W rows into a shared-memory ring with
// 1-D bulk copies (cp.async.bulk + mbarrier transaction counts), so each CTA
// keeps RING rows (48 KB) in flight with no register cost; four consumer warps
// take ring slots round-robin (warp w: owned slots w, w+4, ...), compute the
// dot with the embedding held in registers, the BCE/factor algebra, and
// accumulate f * w_row. The per-warp partials are reduced in warp order
// (deterministic). Replaces the register-pipelined gather (2-3x the HBM rate).
constexpr int kTmaConsumers = 4;
constexpr int kTmaThreads = 32 * (kTmaConsumers + 1);

template <bool BF16>
constexpr int tma_ring() { return BF16 ? 32 : 16; }

template <int NV, bool BF16>
constexpr size_t tma_fwd_smem(int S) {
  return static_cast<size_t>(tma_ring<BF16>()) * NV * 128 * (BF16 ? 2 : 4) + 2 * 8 * tma_ring<BF16>() +
         static_cast<size_t>(S) * 8 + 64;
}

template <int NV, bool BF16>
__global__ void __launch_bounds__(kTmaThreads, 3) slot_forward_tma(FwdArgs a) {
  pdl_entry();
  if (a.skip && *a.skip) return;
  constexpr int d = NV * 128;
  constexpr int RING = tma_ring<BF16>();
  constexpr uint32_t ROWB = d * (BF16 ? 2 : 4);
  extern __shared__ __align__(128) unsigned char fsm[];
  unsigned char* ring = fsm;
  uint64_t* full = reinterpret_cast<uint64_t*>(fsm + RING * ROWB);
  uint64_t* empty = full + RING;
  int32_t* own = reinterpret_cast<int32_t*>(empty + RING);
  __shared__ int s_nown;
  __shared__ double s_loss[kTmaConsumers], s_fabs[kTmaConsumers];
  __shared__ float s_emax[kTmaConsumers];
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* row_ids = a.ids + static_cast<size_t>(b) * a.S;
  // the row's ids -> smem with every thread (independent loads), then warp 0
  // compacts the owned slots in slot order (label-sharded W: others are
  // skipped): own[i] = slot, own_loc[i] = local W row, read by the producer
  // from shared memory (a global load per issued row serialised it).
  int32_t* own_loc = own + a.S;
  for (int sl = threadIdx.x; sl < a.S; sl += kTmaThreads) own_loc[sl] = row_ids[sl];
  __syncthreads();
  if (warp == 0) {
    int n = 0;
    for (int s0 = 0; s0 < a.S; s0 += 32) {
      const int sl = s0 + lane;
      int64_t loc = -1;
      if (sl < a.S) loc = static_cast<int64_t>(own_loc[sl]) - a.off;
      const bool o = loc >= 0 && loc < a.Lloc;
      const unsigned m = __ballot_sync(0xffffffffu, o);
      __syncwarp();  // every lane has read own_loc[s0..s0+31] before it is overwritten below
      if (o) {
        const int at = n + __popc(m & ((1u << lane) - 1u));
        own[at] = sl;
        own_loc[at] = static_cast<int32_t>(loc);
      }
      n += __popc(m);
      __syncwarp();
    }
    if (lane == 0) {
      s_nown = n;
      for (int r = 0; r < RING; ++r) {
        mbar_init(&full[r], 1);
        mbar_init(&empty[r], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  const int n_own = s_nown;
  if (warp == kTmaConsumers) {
    // ---------------- producer
    if (lane == 0) {
      const unsigned char* Wb = static_cast<const unsigned char*>(a.W);
      for (int i = 0; i < n_own; ++i) {
        const int r = i % RING;
        mbar_wait(&empty[r], ((i / RING) & 1) ^ 1);
        mbar_expect_tx(&full[r], ROWB);
        bulk_g2s(ring + r * ROWB, Wb + static_cast<size_t>(own_loc[i]) * ROWB, ROWB, &full[r]);
      }
    }
  } else {
    // ---------------- consumers
    float4 e[NV], g[NV];
    float emax = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      e[i] = *reinterpret_cast<const float4*>(a.emb + static_cast<size_t>(b) * d + i * 128 + lane * 4);
      g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      emax = fmaxf(emax, fmaxf(fmaxf(fabsf(e[i].x), fabsf(e[i].y)), fmaxf(fabsf(e[i].z), fabsf(e[i].w))));
      if (!(isfinite(e[i].x) && isfinite(e[i].y) && isfinite(e[i].z) && isfinite(e[i].w))) emax = INFINITY;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    double lsum = 0.0, fabs_sum = 0.0;
    float pend_sc = 0.0f, pend_pt = 0.0f, pend_wn = 0.0f;  // lane c holds the c-th pending loss term
    int c_pend = 0;
    for (int i = warp; i < n_own; i += kTmaConsumers) {
      const int r = i % RING;
      const int sl = own[i];
      const float fin = a.factors_in ? a.factors_in[static_cast<size_t>(b) * a.S + sl] : 0.0f;
      const SlotMeta meta = slot_meta(a, b, sl);
      mbar_wait(&full[r], (i / RING) & 1);
      float4 w[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        if constexpr (BF16) {
          const uint2 u = *reinterpret_cast<const uint2*>(ring + r * ROWB + (j * 128 + lane * 4) * 2);
          w[j] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                             __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
        } else {
          w[j] = *reinterpret_cast<const float4*>(ring + r * ROWB + (j * 128 + lane * 4) * 4);
        }
      }
      regs_landed(w);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[r]);  // the row is in registers: release the slot
      float f;
      if (a.factors_in) {
        f = fin;
      } else {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          acc = fmaf(w[j].x, e[j].x, acc);
          acc = fmaf(w[j].y, e[j].y, acc);
          acc = fmaf(w[j].z, e[j].z, acc);
          acc = fmaf(w[j].w, e[j].w, acc);
        }
        acc = warp_sum(acc);
        float pt, wn;
        f = slot_factor_meta(meta, acc, &pt, &wn);
        if (lane == c_pend) {
          pend_sc = acc;
          pend_pt = pt;
          pend_wn = wn;
        }
        if (++c_pend == 32) {
          lsum += slot_loss(pend_sc, pend_pt, pend_wn);
          c_pend = 0;
        }
      }
      if (lane == 0) {
        fabs_sum += static_cast<double>(fabsf(f));
        if (a.factors) a.factors[static_cast<size_t>(b) * a.S + sl] = f;
      }
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        g[j].x = fmaf(f, w[j].x, g[j].x);
        g[j].y = fmaf(f, w[j].y, g[j].y);
        g[j].z = fmaf(f, w[j].z, g[j].z);
        g[j].w = fmaf(f, w[j].w, g[j].w);
      }
    }
    if (lane < c_pend) lsum += slot_loss(pend_sc, pend_pt, pend_wn);
    lsum = warp_sum(lsum);
    fabs_sum = warp_sum(fabs_sum);
    if (lane == 0) {
      s_loss[warp] = lsum;
      s_fabs[warp] = fabs_sum;
      s_emax[warp] = emax;
    }
    __syncthreads();  // (1) every ring row consumed: the ring is reused for the partials
    float* red = reinterpret_cast<float*>(ring);
#pragma unroll
    for (int j = 0; j < NV; ++j) *reinterpret_cast<float4*>(red + warp * d + j * 128 + lane * 4) = g[j];
  }
  if (warp == kTmaConsumers) __syncthreads();  // (1), producer side (bar.sync counts threads, not call sites)
  __syncthreads();                             // (2) partials written
  const float* red = reinterpret_cast<const float*>(ring);
  bool bad = false;
  for (int k = threadIdx.x; k < d; k += kTmaThreads) {
    float gk = 0.0f;
#pragma unroll
    for (int w = 0; w < kTmaConsumers; ++w) gk += red[w * d + k];
    if (a.keep) gk = __fmul_rn(gk, a.keep[static_cast<size_t>(b) * d + k]);
    a.grad_emb[static_cast<size_t>(b) * d + k] = gk;
    bad |= !isfinite(gk);
  }
  if (bad) a.status[ASTRA_STATUS_NONFINITE_GRAD_EMB] = 1;
  if (threadIdx.x == 0) {
    double l = 0.0, fa = 0.0;
    for (int w = 0; w < kTmaConsumers; ++w) {
      l += s_loss[w];
      fa += s_fabs[w];
    }
    a.loss_rows[b] = l;
    a.bound_rows[b] = fa * static_cast<double>(s_emax[0]);
  }
}

// Generic forward for any d: emb and the per-warp partials live in shared memory.
template <bool BF16>
__global__ void __launch_bounds__(kFwdThreads) slot_forward_generic(FwdArgs a) {
  pdl_entry();
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(16) float sm[];
  float* e = sm;                 // d
  float* red = sm + a.d;         // kFwdWarps * d
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = a.d;
  __shared__ float s_emax;
  for (int k = threadIdx.x; k < d; k += kFwdThreads) e[k] = a.emb[static_cast<size_t>(b) * d + k];
  for (int k = threadIdx.x; k < kFwdWarps * d; k += kFwdThreads) red[k] = 0.0f;
  __syncthreads();
  if (warp == 0) {
    float m = 0.0f;
    for (int k = lane; k < d; k += 32) m = isfinite(e[k]) ? fmaxf(m, fabsf(e[k])) : INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_emax = m;
  }
  double lsum = 0.0, fabs_sum = 0.0;
  float* gw = red + warp * d;
  for (int s = warp; s < a.S; s += kFwdWarps) {
    int64_t loc = static_cast<int64_t>(a.ids[static_cast<size_t>(b) * a.S + s]) - a.off;
    if (loc < 0 || loc >= a.Lloc) continue;
    float f;
    if (a.factors_in) {
      f = a.factors_in[static_cast<size_t>(b) * a.S + s];
    } else {
      float acc = 0.0f;
      for (int k = lane; k < d; k += 32) {
        size_t el = static_cast<size_t>(loc) * d + k;
        float wv = BF16 ? bf16_bits_to_f32(static_cast<const uint16_t*>(a.W)[el]) : static_cast<const float*>(a.W)[el];
        acc = fmaf(wv, e[k], acc);
      }
      acc = warp_sum(acc);
      double lt;
      f = slot_factor(a, b, s, acc, &lt);
      if (lane == 0) lsum += lt;
    }
    if (lane == 0) {
      fabs_sum += static_cast<double>(fabsf(f));
      if (a.factors) a.factors[static_cast<size_t>(b) * a.S + s] = f;
    }
    for (int k = lane; k < d; k += 32) {
      size_t el = static_cast<size_t>(loc) * d + k;
      float wv = BF16 ? bf16_bits_to_f32(static_cast<const uint16_t*>(a.W)[el]) : static_cast<const float*>(a.W)[el];
      gw[k] = fmaf(f, wv, gw[k]);
    }
  }
  __syncthreads();
  forward_tail(a, b, red, lsum, fabs_sum, s_emax);
}

// Fixed-order fp64 sums of the per-row loss and overflow bound.
__global__ void __launch_bounds__(1024) finalize_kernel(const double* loss_rows, const double* bound_rows, int B,
                                                        double* loss_out, int32_t* status) {
  pdl_entry();
  __shared__ double sl[1024], sb[1024];
  double l = 0.0, bd = 0.0;
  for (int i = threadIdx.x; i < B; i += 1024) {
    l += loss_rows[i];
    bd += bound_rows[i];
  }
  sl[threadIdx.x] = l;
  sb[threadIdx.x] = bd;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sl[threadIdx.x] += sl[threadIdx.x + o];
      sb[threadIdx.x] += sb[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *loss_out = sl[0];
    if (!(sb[0] < kBoundSafe)) status[ASTRA_STATUS_BOUND_UNSAFE] = 1;
  }
}

// ---------------------------------------------------------------- counting sort

__device__ __forceinline__ float absmax4(float4 v) {
  return fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
}

// Also (sf_acc != null, the single-pass schedule) the finiteness bounds:
// sum over owned slots of (1 + |weight|) and max|emb| (+inf if non-finite).
__global__ void __launch_bounds__(256) count_kernel(const int32_t* ids, int64_t n, int64_t off, int64_t Lloc,
                                                    uint32_t* counts, int32_t* rank, int32_t* status,
                                                    const float* weights, int64_t wstride, int S, const float* emb,
                                                    int64_t n_emb, double* sf_acc, unsigned* emax_acc,
                                                    float* zero_out) {
  pdl_entry();
  if (zero_out) {  // (n_emb floats, 16-byte aligned on the single-pass path)
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_emb / 4;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
      reinterpret_cast<float4*>(zero_out)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  double sf = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t id = ids[i];
    if (id < 0) status[ASTRA_STATUS_ID_RANGE] = 1;
    int64_t loc = static_cast<int64_t>(id) - off;
    const bool own = loc >= 0 && loc < Lloc;
    rank[i] = own ? static_cast<int32_t>(atomicAdd(counts + loc, 1u)) : -1;
    if (sf_acc && own) {
      const int b = static_cast<int>(i) / S;  // (n < 2^31)
      const float wt = weights[b * wstride + (static_cast<int>(i) - b * S)];
      sf += 1.0 + (isfinite(wt) ? fabs(static_cast<double>(wt)) : INFINITY);
    }
  }
  if (!sf_acc) return;
  float em = 0.0f;
  // (n_emb % 4 == 0 and emb 16-byte aligned on the single-pass path)
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_emb / 4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 e = reinterpret_cast<const float4*>(emb)[i];
    const bool fin = isfinite(e.x) && isfinite(e.y) && isfinite(e.z) && isfinite(e.w);
    em = fmaxf(em, fin ? absmax4(e) : INFINITY);
  }
  __shared__ double s_sf[8];
  __shared__ float s_em[8];
  sf = warp_sum(sf);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) em = fmaxf(em, __shfl_xor_sync(0xffffffffu, em, o));
  if ((threadIdx.x & 31) == 0) {
    s_sf[threadIdx.x >> 5] = sf;
    s_em[threadIdx.x >> 5] = em;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    float m = 0.0f;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      t += s_sf[w];
      m = fmaxf(m, s_em[w]);
    }
    if (t != 0.0) atomicAdd(sf_acc, t);
    atomicMax(emax_acc, __float_as_uint(m));  // non-negative floats order as their bits
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* counts, int64_t Lloc,
                                                                   uint32_t* blk_slots, uint32_t* blk_nz) {
  pdl_entry();
  __shared__ uint32_t ss[kScanThreads / 32], sn[kScanThreads / 32];
  int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  uint32_t s = 0, nz = 0;
  for (int i = 0; i < kScanItems; ++i) {
    int64_t l = base + i * kScanThreads + threadIdx.x;
    if (l < Lloc) {
      uint32_t c = counts[l];
      s += c;
      nz += c > 0;
    }
  }
  s = warp_sum(s);
  nz = warp_sum(nz);
  if ((threadIdx.x & 31) == 0) {
    ss[threadIdx.x >> 5] = s;
    sn[threadIdx.x >> 5] = nz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t a = 0, c = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) {
      a += ss[w];
      c += sn[w];
    }
    blk_slots[blockIdx.x] = a;
    blk_nz[blockIdx.x] = c;
  }
}

// Exclusive scan of the per-block sums (single CTA), writes U.
// (mode != null: also decides the step schedule from count_kernel's bounds.)
__global__ void __launch_bounds__(1024) scan_top_kernel(uint32_t* blk_slots, uint32_t* blk_nz, int nb,
                                                        uint32_t* U, const double* sf_acc, const unsigned* emax_acc,
                                                        const float* w_absmax, int32_t* mode, int d) {
  pdl_entry();
  __shared__ uint32_t cs[1024], cn[1024];
  const int per = (nb + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(nb, lo + per);
  uint32_t a = 0, c = 0;
  for (int i = lo; i < hi; ++i) {
    a += blk_slots[i];
    c += blk_nz[i];
  }
  cs[threadIdx.x] = a;
  cn[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    uint32_t xa = threadIdx.x >= o ? cs[threadIdx.x - o] : 0;
    uint32_t xc = threadIdx.x >= o ? cn[threadIdx.x - o] : 0;
    __syncthreads();
    cs[threadIdx.x] += xa;
    cn[threadIdx.x] += xc;
    __syncthreads();
  }
  uint32_t ra = cs[threadIdx.x] - a, rc = cn[threadIdx.x] - c;  // exclusive
  for (int i = lo; i < hi; ++i) {
    uint32_t va = blk_slots[i], vc = blk_nz[i];
    blk_slots[i] = ra;
    blk_nz[i] = rc;
    ra += va;
    rc += vc;
  }
  if (threadIdx.x == 1023) *U = cn[1023];
  if (mode && threadIdx.x == 0) {
    const double SF = *sf_acc;
    const float EM = __uint_as_float(*emax_acc);
    const float WM = w_absmax ? *w_absmax : INFINITY;
    // every gradient entry <= SF * EM, every grad_emb entry <= SF * WM, and
    // every partial sum of a score's dot product <= d * EM * WM (no fp32
    // overflow -> inf - inf = NaN in a score, which no later check would see)
    *mode = isfinite(SF) && isfinite(EM) && isfinite(WM) && SF * static_cast<double>(EM) < kSingleSafe &&
            SF * static_cast<double>(WM) < kSingleSafe &&
            static_cast<double>(d) * static_cast<double>(EM) * static_cast<double>(WM) < kSingleSafe;
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const uint32_t* counts, int64_t Lloc,
                                                                  const uint32_t* blk_slots,
                                                                  const uint32_t* blk_nz, uint32_t* offsets,
                                                                  int32_t* uniq, uint32_t* ustart, uint32_t* ucnt,
                                                                  uint32_t* n_hot = nullptr, int32_t* hot_u = nullptr) {
  pdl_entry();
  __shared__ uint32_t ws[kScanThreads / 32], wn[kScanThreads / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanItems;
  uint32_t c[kScanItems];
  uint32_t s = 0, nz = 0;
  if (base + kScanItems <= Lloc) {  // full run: 16-byte loads (workspace arrays are 256-byte aligned)
#pragma unroll
    for (int i = 0; i < kScanItems; i += 4) {
      const uint4 v = *reinterpret_cast<const uint4*>(counts + base + i);
      c[i] = v.x;
      c[i + 1] = v.y;
      c[i + 2] = v.z;
      c[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) c[i] = base + i < Lloc ? counts[base + i] : 0u;
  }
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    s += c[i];
    nz += c[i] > 0;
  }
  // block-exclusive scan of (s, nz) over threads
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t is = s, in = nz;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t xs = __shfl_up_sync(0xffffffffu, is, o), xn = __shfl_up_sync(0xffffffffu, in, o);
    if (lane >= o) {
      is += xs;
      in += xn;
    }
  }
  if (lane == 31) {
    ws[warp] = is;
    wn[warp] = in;
  }
  __syncthreads();
  uint32_t ps = blk_slots[blockIdx.x], pn = blk_nz[blockIdx.x];
  for (int w = 0; w < warp; ++w) {
    ps += ws[w];
    pn += wn[w];
  }
  ps += is - s;
  pn += in - nz;
  uint32_t o[kScanItems];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t l = base + i;
    o[i] = ps;
    if (l < Lloc) {
      if (c[i]) {
        uniq[pn] = static_cast<int32_t>(l);
        if (ustart) {
          ustart[pn] = ps;
          ucnt[pn] = c[i];
          if (hot_u && is_hot(c[i])) hot_u[atomicAdd(n_hot, 1u)] = static_cast<int32_t>(pn);
        }
        ++pn;
      }
      ps += c[i];
    }
  }
  if (base + kScanItems <= Lloc) {
#pragma unroll
    for (int i = 0; i < kScanItems; i += 4)
      *reinterpret_cast<uint4*>(offsets + base + i) = make_uint4(o[i], o[i + 1], o[i + 2], o[i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
      if (base + i < Lloc) offsets[base + i] = o[i];
  }
}

__global__ void scatter_kernel(const int32_t* ids, const int32_t* rank, int64_t n, int64_t off,
                               const uint32_t* offsets, int32_t* perm) {
  pdl_entry();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t r = rank[i];
    if (r >= 0) perm[offsets[static_cast<int64_t>(ids[i]) - off] + r] = static_cast<int32_t>(i);
  }
}

// ---------------------------------------------------------------- label-major update

struct UpdArgs {
  const float* emb;
  const float* factors;
  const int32_t* uniq;
  const uint32_t* U;
  const uint32_t* offsets;
  const uint32_t* counts;
  const int32_t* perm;
  int32_t* perm2;  // sorted segments longer than 32
  int S, d;
  void* W;
  float* m;
  float* v;
  float lr, wd;
  float c1, c2, eps, neg_step;  // Adam: fp32(1-b1), fp32(1-b2), eps, fp32(-lr*sqrt(bc2)/bc1)
  int32_t* status;
  float* w_absmax;  // running max|W| bound kept current by every update kernel (or null)
  const int32_t* skip = nullptr;  // as FwdArgs::skip
};

// Fold a warp's max |new W| into the running bound (non-negative floats order as bits).
__device__ __forceinline__ void push_wmax(const UpdArgs& a, float wmax, int lane) {
  if (!a.w_absmax) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
  if (lane == 0 && wmax > 0.0f) atomicMax(reinterpret_cast<unsigned*>(a.w_absmax), __float_as_uint(wmax));
}


// Sort the label's slot indices ascending. Segments <= 32 stay in a register
// (returned); longer ones are rank-sorted into perm2.
__device__ __forceinline__ int32_t sort_segment(const UpdArgs& a, uint32_t start, uint32_t n, int lane) {
  if (n <= 2) {  // (most multi-occurrence labels: one compare-exchange)
    int32_t v = lane < static_cast<int>(n) ? a.perm[start + lane] : INT_MAX;
    const int32_t o = __shfl_xor_sync(0xffffffffu, v, 1);
    return lane == 0 ? min(v, o) : (lane == 1 ? max(v, o) : v);
  }
  if (n <= 32) {
    int32_t v = lane < static_cast<int>(n) ? a.perm[start + lane] : INT_MAX;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        int32_t o = __shfl_xor_sync(0xffffffffu, v, stride);
        bool up = (lane & size) == 0;
        bool lower = (lane & stride) == 0;
        int32_t lo = min(v, o), hi = max(v, o);
        v = (lower == up) ? lo : hi;
      }
    }
    return v;
  }
  for (uint32_t i = lane; i < n; i += 32) {
    int32_t x = a.perm[start + i];
    uint32_t r = 0;
    for (uint32_t j = 0; j < n; ++j) r += a.perm[start + j] < x;
    a.perm2[start + r] = x;
  }
  __syncwarp();
  return 0;
}

__device__ __forceinline__ int32_t seg_slot(const UpdArgs& a, uint32_t start, uint32_t n, int32_t reg, uint32_t j) {
  return n <= 32 ? __shfl_sync(0xffffffffu, reg, static_cast<int>(j)) : a.perm2[start + j];
}

#ifndef ASTRA_ADAM_FAST
#define ASTRA_ADAM_FAST 1
#endif
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// One element's update: SGD (classifiers.py:82, each op rounded like NumPy)
// or SparseAdam (torch.optim.SparseAdam op order).
// FAST (Adam on bf16 W, ASTRA_ADAM_FAST): MUFU sqrt + reciprocal (each ~1
// ulp) instead of the IEEE sqrt/div sequences; the step term then differs from
// SparseAdam's by a few ulp of itself, far below the bf16 rounding of W'.
template <bool ADAM, bool FAST = false>
__device__ __forceinline__ float upd_elem(const UpdArgs& a, float p, float g, float* mp, float* vp) {
  if constexpr (!ADAM) {
    return __fsub_rn(p, __fmul_rn(a.lr, __fadd_rn(g, __fmul_rn(a.wd, p))));
  } else {
    if (a.wd != 0.0f) g = __fadd_rn(g, __fmul_rn(a.wd, p));
    float m0 = *mp, v0 = *vp;
    float mu = __fmul_rn(__fsub_rn(g, m0), a.c1);
    float vu = __fmul_rn(__fsub_rn(__fmul_rn(g, g), v0), a.c2);
    *mp = __fadd_rn(m0, mu);
    *vp = __fadd_rn(v0, vu);
    float numer = __fadd_rn(mu, m0);
    if constexpr (FAST) {
      const float denom = __fadd_rn(sqrt_approx(__fadd_rn(vu, v0)), a.eps);
      return __fadd_rn(p, __fmul_rn(a.neg_step, __fmul_rn(numer, rcp_approx(denom))));
    } else {
      const float denom = __fadd_rn(__fsqrt_rn(__fadd_rn(vu, v0)), a.eps);
      return __fadd_rn(p, __fmul_rn(a.neg_step, __fdiv_rn(numer, denom)));
    }
  }
}

template <bool BF16>
__device__ __forceinline__ float load_p(const void* W, size_t el) {
  return BF16 ? bf16_bits_to_f32(static_cast<const uint16_t*>(W)[el]) : static_cast<const float*>(W)[el];
}
template <bool BF16>
__device__ __forceinline__ void store_p(void* W, size_t el, float v) {
  if constexpr (BF16)
    static_cast<uint16_t*>(W)[el] = f32_to_bf16_bits(v);
  else
    static_cast<float*>(W)[el] = v;
}

// CHECK_ONLY: compute every gradient, flag non-finite ones, write nothing.
template <bool BF16, bool ADAM, bool CHECK_ONLY>
__global__ void __launch_bounds__(kUpdThreads) label_update_kernel(UpdArgs a) {
  pdl_entry();
  if (a.skip && *a.skip) return;
  const int lane = threadIdx.x & 31;
  if (CHECK_ONLY) {
    if (!a.status[ASTRA_STATUS_BOUND_UNSAFE]) return;  // finiteness already proven
  } else {
    if (a.status[ASTRA_STATUS_NONFINITE_GRAD_EMB] || a.status[ASTRA_STATUS_NONFINITE_GRAD]) return;
  }
  const uint32_t U = *a.U;
  const int d = a.d;
  const uint32_t warps = gridDim.x * (kUpdThreads / 32);
  float wmax = 0.0f;
  for (uint32_t u = blockIdx.x * (kUpdThreads / 32) + (threadIdx.x >> 5); u < U; u += warps) {
    const int32_t l = a.uniq[u];
    const uint32_t start = a.offsets[l], n = a.counts[l];
    const int32_t reg = sort_segment(a, start, n, lane);
    bool bad = false;
    for (int k0 = 0; k0 < d; k0 += 128) {
      // each lane: 4 consecutive elements of this 128-wide chunk
      const int k = k0 + lane * 4;
      float g[4] = {0.f, 0.f, 0.f, 0.f};
      const int nk = k < d ? min(4, d - k) : 0;
      for (uint32_t j = 0; j < n; ++j) {
        const int32_t slot = seg_slot(a, start, n, reg, j);
        const float f = a.factors[slot];
        const float* e = a.emb + static_cast<size_t>(slot / a.S) * d + k;
        for (int t = 0; t < nk; ++t) g[t] = __fadd_rn(g[t], __fmul_rn(f, e[t]));
      }
      for (int t = 0; t < nk; ++t) bad |= !isfinite(g[t]);
      if (!CHECK_ONLY) {
        const size_t row = static_cast<size_t>(l) * d;
        for (int t = 0; t < nk; ++t) {
          float p = load_p<BF16>(a.W, row + k + t);
          float np = upd_elem<ADAM>(a, p, g[t], ADAM ? a.m + row + k + t : nullptr, ADAM ? a.v + row + k + t : nullptr);
          store_p<BF16>(a.W, row + k + t, np);
          wmax = fmaxf(wmax, fabsf(np));
        }
      }
    }
    if (CHECK_ONLY && __any_sync(0xffffffffu, bad)) a.status[ASTRA_STATUS_NONFINITE_GRAD] = 1;
  }
  if (!CHECK_ONLY) push_wmax(a, wmax, lane);
}

// TMA-fed SGD update (the default for d % 128 == 0): each CTA owns a
// contiguous chunk of the sorted unique-label list; one producer lane streams
// the chunk's W rows into a shared-memory ring with bulk copies while four
// consumer warps (warp w: the chunk's labels w, w+4, ...) sum the label's
// gradient from the L2-resident embeddings (same ascending-slot order and
// roundings as label_update_kernel), then take the row from the ring, apply the
// update and store it. W is read and written once per touched row.
// Ring geometry of the update: one entry = the W row (+ the Adam m and v rows).
#ifndef ASTRA_UPD_ADAM_RING
#define ASTRA_UPD_ADAM_RING 8
#endif
template <int NV, bool BF16, bool ADAM>
struct UpdRing {
  static constexpr uint32_t WB = NV * 128 * (BF16 ? 2 : 4);
  static constexpr uint32_t MB = ADAM ? NV * 128 * 4 : 0;
  static constexpr uint32_t ENTRY = WB + 2 * MB;
  static constexpr int RING = ADAM ? ASTRA_UPD_ADAM_RING : (BF16 ? 32 : 16);
  static constexpr size_t smem() { return static_cast<size_t>(RING) * ENTRY + 2 * 8 * RING; }
};

// CTAs per SM of the TMA update: three (Adam too: 124 registers and an
// 8 x 9 KB ring fit; 1.31 vs 1.67 ms per minibatch at 2 for bf16 Adam), except
// Adam at d = 1024, whose moments spill at three.
#ifndef ASTRA_UPD_ADAM_CTAS
#define ASTRA_UPD_ADAM_CTAS 3
#endif
template <int NV, bool ADAM>
constexpr int upd_tma_ctas() { return ADAM && NV > 6 ? 2 : (ADAM ? ASTRA_UPD_ADAM_CTAS : 3); }

template <int NV, bool BF16, bool ADAM>
__global__ void __launch_bounds__(kTmaThreads, upd_tma_ctas<NV, ADAM>()) label_update_tma(UpdArgs a) {
  pdl_entry();
  if (a.skip && *a.skip) return;
  constexpr int d = NV * 128;
  using RG = UpdRing<NV, BF16, ADAM>;
  constexpr int RING = RG::RING;
  constexpr uint32_t ROWB = RG::ENTRY;
  extern __shared__ __align__(128) unsigned char usm[];
  unsigned char* ring = usm;
  uint64_t* full = reinterpret_cast<uint64_t*>(usm + RING * ROWB);
  uint64_t* empty = full + RING;
  if (a.status[ASTRA_STATUS_NONFINITE_GRAD_EMB] || a.status[ASTRA_STATUS_NONFINITE_GRAD]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t U = *a.U;
  const uint32_t chunk = (U + gridDim.x - 1) / gridDim.x;
  const uint32_t u0 = min(U, blockIdx.x * chunk), u1 = min(U, u0 + chunk);
  const int n_mine = static_cast<int>(u1 - u0);
  if (n_mine == 0) return;
  if (threadIdx.x == 0) {
    for (int r = 0; r < RING; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kTmaConsumers) {
    // producer warp: 32 label ids per coalesced load, lane 0 issues the copies
    const unsigned char* Wb = static_cast<const unsigned char*>(a.W);
    for (int i0 = 0; i0 < n_mine; i0 += 32) {
      const int32_t l_lane = i0 + lane < n_mine ? a.uniq[u0 + i0 + lane] : 0;
      const int nb = min(32, n_mine - i0);
      for (int jj = 0; jj < nb; ++jj) {
        const size_t l = static_cast<size_t>(__shfl_sync(0xffffffffu, l_lane, jj));
        if (lane == 0) {
          const int i = i0 + jj, r = i % RING;
          mbar_wait(&empty[r], ((i / RING) & 1) ^ 1);
          mbar_expect_tx(&full[r], ROWB);
          unsigned char* dst = ring + r * ROWB;
          bulk_g2s(dst, Wb + l * RG::WB, RG::WB, &full[r]);
          if constexpr (ADAM) {
            bulk_g2s(dst + RG::WB, a.m + l * d, RG::MB, &full[r]);
            bulk_g2s(dst + RG::WB + RG::MB, a.v + l * d, RG::MB, &full[r]);
          }
        }
        __syncwarp();
      }
    }
    return;
  }
  float wmax = 0.0f;
  for (int i = warp; i < n_mine; i += kTmaConsumers) {
    const int r = i % RING;
    const int32_t l = a.uniq[u0 + i];
    const uint32_t start = a.offsets[l], n = a.counts[l];
    const int32_t reg = sort_segment(a, start, n, lane);
    const size_t row = static_cast<size_t>(l) * d;
    float4 g[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) g[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t j = 0;
    for (; j + 2 <= n; j += 2) {  // two occurrences' loads in flight, summed in order
      const int32_t s0 = seg_slot(a, start, n, reg, j), s1 = seg_slot(a, start, n, reg, j + 1);
      const float f0 = a.factors[s0], f1 = a.factors[s1];
      const float* e0 = a.emb + static_cast<size_t>(s0 / a.S) * d + lane * 4;
      const float* e1 = a.emb + static_cast<size_t>(s1 / a.S) * d + lane * 4;
      float4 x0[NV], x1[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        x0[q] = *reinterpret_cast<const float4*>(e0 + q * 128);
        x1[q] = *reinterpret_cast<const float4*>(e1 + q * 128);
      }
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        g[q].x = __fadd_rn(g[q].x, __fmul_rn(f0, x0[q].x));
        g[q].y = __fadd_rn(g[q].y, __fmul_rn(f0, x0[q].y));
        g[q].z = __fadd_rn(g[q].z, __fmul_rn(f0, x0[q].z));
        g[q].w = __fadd_rn(g[q].w, __fmul_rn(f0, x0[q].w));
        g[q].x = __fadd_rn(g[q].x, __fmul_rn(f1, x1[q].x));
        g[q].y = __fadd_rn(g[q].y, __fmul_rn(f1, x1[q].y));
        g[q].z = __fadd_rn(g[q].z, __fmul_rn(f1, x1[q].z));
        g[q].w = __fadd_rn(g[q].w, __fmul_rn(f1, x1[q].w));
      }
    }
    if (j < n) {
      const int32_t s0 = seg_slot(a, start, n, reg, j);
      const float f0 = a.factors[s0];
      const float* e0 = a.emb + static_cast<size_t>(s0 / a.S) * d + lane * 4;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const float4 x0 = *reinterpret_cast<const float4*>(e0 + q * 128);
        g[q].x = __fadd_rn(g[q].x, __fmul_rn(f0, x0.x));
        g[q].y = __fadd_rn(g[q].y, __fmul_rn(f0, x0.y));
        g[q].z = __fadd_rn(g[q].z, __fmul_rn(f0, x0.z));
        g[q].w = __fadd_rn(g[q].w, __fmul_rn(f0, x0.w));
      }
    }
    mbar_wait(&full[r], (i / RING) & 1);
    float4 p[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      if constexpr (BF16) {
        const uint2 u = *reinterpret_cast<const uint2*>(ring + r * ROWB + (q * 128 + lane * 4) * 2);
        p[q] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                           __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
      } else {
        p[q] = *reinterpret_cast<const float4*>(ring + r * ROWB + (q * 128 + lane * 4) * 4);
      }
    }
    float4 m4[ADAM ? NV : 1], v4[ADAM ? NV : 1];
    if constexpr (ADAM) {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        m4[q] = *reinterpret_cast<const float4*>(ring + r * ROWB + RG::WB + (q * 128 + lane * 4) * 4);
        v4[q] = *reinterpret_cast<const float4*>(ring + r * ROWB + RG::WB + RG::MB + (q * 128 + lane * 4) * 4);
      }
      regs_landed(m4);
      regs_landed(v4);
    }
    regs_landed(p);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[r]);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      float4 np;
      const size_t el = row + q * 128 + lane * 4;
      if constexpr (ADAM) {
        np.x = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p[q].x, g[q].x, &m4[q].x, &v4[q].x);
        np.y = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p[q].y, g[q].y, &m4[q].y, &v4[q].y);
        np.z = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p[q].z, g[q].z, &m4[q].z, &v4[q].z);
        np.w = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p[q].w, g[q].w, &m4[q].w, &v4[q].w);
        *reinterpret_cast<float4*>(a.m + el) = m4[q];
        *reinterpret_cast<float4*>(a.v + el) = v4[q];
      } else {
        np.x = upd_elem<false>(a, p[q].x, g[q].x, nullptr, nullptr);
        np.y = upd_elem<false>(a, p[q].y, g[q].y, nullptr, nullptr);
        np.z = upd_elem<false>(a, p[q].z, g[q].z, nullptr, nullptr);
        np.w = upd_elem<false>(a, p[q].w, g[q].w, nullptr, nullptr);
      }
      if constexpr (BF16) {
        uint2 o;
        o.x = static_cast<uint32_t>(f32_to_bf16_bits(np.x)) | (static_cast<uint32_t>(f32_to_bf16_bits(np.y)) << 16);
        o.y = static_cast<uint32_t>(f32_to_bf16_bits(np.z)) | (static_cast<uint32_t>(f32_to_bf16_bits(np.w)) << 16);
        *reinterpret_cast<uint2*>(static_cast<uint16_t*>(a.W) + el) = o;
      } else {
        *reinterpret_cast<float4*>(static_cast<float*>(a.W) + el) = np;
      }
      wmax = fmaxf(wmax, absmax4(np));  // (bf16: the bound holds for the rounded value too)
    }
  }
  push_wmax(a, wmax, lane);
}

// ================================================================ single-pass step
// The default schedule (SGD and Adam; ASTRA_STEP_SINGLE_ADAM=0: Adam two-kernel) when
// d % 128 == 0, d <= 768: ONE label-major pass over the touched rows. Each CTA
// owns a contiguous chunk of the sorted unique-label list; a producer warp
// builds each label's descriptor (bucket, first occurrence + its metadata)
// into an in-order queue and bulk-copies the W row (+ Adam m, v) into any free
// data slot of a shared-memory pool; consumer warp w takes labels w, w+4, ...,
// pulling the next label's embedding row towards L1 first. For label l
// it holds the OLD row in registers and walks l's slots in ascending b*S+s
// order: score = <emb_b, W_l> (the forward's fma order and butterfly, so the
// same bits), factor (trainer.py:369-380), g += f * emb_b (label_update's
// order and roundings, so W' is bit-identical to the two-kernel schedule), and
// grad_emb[b] += f * W_l (vector fp32 reductions into the L2-resident B x d
// buffer, red.global.add.v4.f32); then it writes the updated row. DRAM sees
// each touched row read once and written once (U*d*(2*w_W + 2*s_opt)), instead
// of the gather's extra B*S*d*w_W read.
//
// Finiteness (classifiers.py:79-80: nothing is written when a gradient is
// non-finite) is proven before the pass from bounds that need no scores:
// S_f = sum over owned slots of (1 + |weight|) >= sum |factor|, so every label
// gradient is <= S_f * max|emb| and every grad_emb entry <= S_f * max|W|
// (max|W|: the running bound w_absmax). count_kernel accumulates S_f and
// max|emb|, scan_top_kernel decides (mode = 1: this pass; 0: the two-kernel
// schedule, whose kernels are launched too and return at once when mode = 1).
// grad_emb's summation order over slots follows the reduction order, so it is
// not bitwise run-to-run deterministic (astra_set_step_deterministic(1) or
// ASTRA_STEP_SINGLE=0 select the deterministic two-kernel schedule); the fp64
// loss terms are evaluated lane-parallel in the pass and reduced per row in slot
// order by single_row_finalize from the stored per-slot fp64 loss terms.
struct SingleArgs {
  FwdArgs f;
  UpdArgs u;
  double* slot_loss;      // [B*S] fp64 loss term of every owned slot
  const int32_t* mode;    // decided by scan_top_kernel
  const uint32_t* ustart; // [U] bucket start of unique label u (= offsets[uniq[u]])
  const uint32_t* ucnt;   // [U] its occurrence count
};

__device__ __forceinline__ void red_add_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

template <int NV>
__device__ __forceinline__ void load_emb_row(const float* emb, int b, int lane, float4 (&e)[NV]) {
  const float* p = emb + static_cast<size_t>(b) * (NV * 128) + lane * 4;
#pragma unroll
  for (int q = 0; q < NV; ++q) e[q] = *reinterpret_cast<const float4*>(p + q * 128);
}

#ifndef ASTRA_SINGLE_CTAS
#define ASTRA_SINGLE_CTAS 4
#endif
#ifndef ASTRA_SINGLE_POLL_NS
#define ASTRA_SINGLE_POLL_NS 20  // producer's back-off while every ring slot is busy
#endif
#ifndef ASTRA_SINGLE_ADAM_EARLY
#define ASTRA_SINGLE_ADAM_EARLY 1  // Adam: moments into registers with the row, ring entry released at once
#endif
#ifndef ASTRA_SINGLE_ADAM_CTAS
#define ASTRA_SINGLE_ADAM_CTAS 2
#endif
// Ring geometry of the single pass: one entry = the W row (+ Adam m, v), and a
// 32-byte descriptor per entry written by the producer (its own barrier, so a
// consumer reads it before the row lands and prefetches the embedding rows).
template <int NV, bool BF16, bool ADAM>
struct SingleRing {
  static constexpr uint32_t WB = NV * 128 * (BF16 ? 2 : 4);
  static constexpr uint32_t MB = ADAM ? NV * 128 * 4 : 0;
  static constexpr uint32_t ENTRY = WB + 2 * MB;
  static constexpr uint32_t SCRATCH = kTmaConsumers * NV * 128 * 4;  // per-warp gradient of multi-slot labels
  static constexpr int Q = 64;                                        // in-order label queue (descriptors)
  static constexpr uint32_t QBYTES = Q * (48 + 16);
  static constexpr int CTAS = ADAM ? ASTRA_SINGLE_ADAM_CTAS : ASTRA_SINGLE_CTAS;
  static constexpr uint32_t BUDGET = (ADAM ? (ASTRA_SINGLE_ADAM_CTAS == 3 ? 74u : 110u)
                                           : (ASTRA_SINGLE_CTAS == 5 ? 44u : 56u)) * 1024;
  static constexpr int RING_MAX = static_cast<int>((BUDGET - SCRATCH - QBYTES) / (ENTRY + 16));
  static constexpr int RING = RING_MAX > 32 ? 32 : RING_MAX;
  static constexpr size_t smem() { return static_cast<size_t>(RING) * (ENTRY + 16) + SCRATCH + QBYTES + 16; }
};

// The producer's per-label descriptor: bucket, first occurrence and its metadata.
struct SingleDesc {
  int32_t l;
  uint32_t start, n;
  int32_t slot0;
  float yf0, w0;
  int32_t o0;
  int32_t pad;
};

// A queue entry: the label's descriptor + the data slot its rows went to and
// the parity of that fill.
struct SingleQEntry {
  SingleDesc dc;
  uint32_t slot, fpar;
  uint32_t pad[2];
};

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Pull a d-float embedding row into L1 (lane i: its 128-byte line(s)).
template <int NV>
__device__ __forceinline__ void prefetch_emb_l1(const float* emb, int b, int lane) {
  const char* row = reinterpret_cast<const char*>(emb + static_cast<size_t>(b) * (NV * 128));
  for (int c = lane; c < NV * 4; c += 32) asm volatile("prefetch.global.L1 [%0];" ::"l"(row + c * 128));
}

template <int NV, bool BF16, bool ADAM>
__global__ void __launch_bounds__(kTmaThreads, SingleRing<NV, BF16, ADAM>::CTAS) step_single_tma(SingleArgs A) {
  pdl_entry();
  constexpr int d = NV * 128;
  using RG = SingleRing<NV, BF16, ADAM>;
  constexpr int RING = RG::RING;
  constexpr int Q = RG::Q;
  constexpr uint32_t ROWB = RG::ENTRY;
  extern __shared__ __align__(128) unsigned char usm[];
  // [RING data slots][queue entries][per-warp scratch][barriers]
  unsigned char* ring = usm;
  SingleQEntry* queue = reinterpret_cast<SingleQEntry*>(usm + RING * ROWB);
  float* gs_all = reinterpret_cast<float*>(queue + Q);
  uint64_t* full = reinterpret_cast<uint64_t*>(gs_all + kTmaConsumers * d);
  uint64_t* empty = full + RING;
  uint64_t* qfull = empty + RING;
  uint64_t* qempty = qfull + Q;
  // free data slots (bit r: slot r released by its consumer): a hint that
  // spares the producer polling every slot's barrier; the barrier stays the
  // synchronisation (the producer still waits on it, which then passes at once)
  uint32_t* freemask = reinterpret_cast<uint32_t*>(qempty + Q);
  if (!*A.mode) return;
  const UpdArgs& a = A.u;
  const FwdArgs& fa = A.f;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t U = *a.U;
  const uint32_t chunk = (U + gridDim.x - 1) / gridDim.x;
  const uint32_t u0 = min(U, blockIdx.x * chunk), u1 = min(U, u0 + chunk);
  const int n_mine = static_cast<int>(u1 - u0);
  if (n_mine == 0) return;
  if (threadIdx.x == 0) {
    for (int r = 0; r < RING; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], 1);
    }
    for (int r = 0; r < Q; ++r) {
      mbar_init(&qfull[r], 1);
      mbar_init(&qempty[r], 1);
    }
    *freemask = RING == 32 ? 0xFFFFFFFFu : ((1u << RING) - 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int S = fa.S;
  auto release = [&](int r) {  // lane 0, after __syncwarp: the slot's reads are done
    mbar_arrive(&empty[r]);
    atomicOr(freemask, 1u << r);
  };
  if (warp == kTmaConsumers) {
    // producer warp: 32 labels per batch, every index load lane-parallel and
    // software-pipelined over batches (batch k+3: bucket, k+2: first
    // occurrence, k+1: its metadata). Labels enter an in-order queue of
    // descriptors; their rows (W, Adam moments) go to ANY free data slot (a
    // slow label holds only its own slot, not the ring), the slot and its fill
    // parity travel in the queue entry.
    const unsigned char* Wb = static_cast<const unsigned char*>(a.W);
    struct PIdx {
      int32_t l;
      uint32_t start, n;
      int32_t slot0;
    };
    auto idx_load = [&](int i0, PIdx& q) {
      q.l = 0;
      q.start = q.n = 0;
      q.slot0 = 0;
      if (i0 + lane < n_mine) {
        const uint32_t u = u0 + i0 + lane;
        q.l = a.uniq[u];
        q.start = A.ustart[u];
        q.n = A.ucnt[u];
      }
    };
    auto perm_load = [&](int i0, PIdx& q) {
      if (i0 + lane < n_mine) q.slot0 = a.perm[q.start];
    };
    auto meta_load = [&](int i0, const PIdx& q, SingleDesc& dl) {
      dl.l = q.l;
      dl.start = q.start;
      dl.n = q.n;
      dl.slot0 = q.slot0;
      dl.yf0 = dl.w0 = 0.0f;
      dl.o0 = 0;
      dl.pad = 0;
      if (i0 + lane < n_mine) {
        const int b0 = q.slot0 / S;
        const SlotMeta m = slot_meta(fa, b0, q.slot0 - b0 * S);
        dl.yf0 = m.yf;
        dl.w0 = m.w;
        dl.o0 = m.o;
      }
    };
    PIdx q1, q2, q3;
    SingleDesc cur;
    idx_load(0, q1);
    perm_load(0, q1);
    meta_load(0, q1, cur);
    idx_load(32, q1);
    perm_load(32, q1);
    idx_load(64, q2);
    uint32_t use = 0;  // bit s: parity of the number of fills of data slot s
    for (int i0 = 0; i0 < n_mine; i0 += 32) {
      SingleDesc nxt;
      meta_load(i0 + 32, q1, nxt);
      perm_load(i0 + 64, q2);
      idx_load(i0 + 96, q3);
      const int nb = min(32, n_mine - i0);
      for (int jj = 0; jj < nb; ++jj) {
        const int i = i0 + jj, qi = i % Q;
        // a hot label takes a queue entry (its consumer skips it) but no data slot
        const bool hot = is_hot(__shfl_sync(0xffffffffu, cur.n, jj));
        int sl = -1;
        if (lane == 0) {
          mbar_wait(&qempty[qi], ((i / Q) & 1) ^ 1);
          if (!hot) {
            uint32_t m;  // a free data slot: its previous fill released
            while ((m = *reinterpret_cast<volatile uint32_t*>(freemask)) == 0u) __nanosleep(ASTRA_SINGLE_POLL_NS);
            sl = __ffs(m) - 1;
            atomicAnd(freemask, ~(1u << sl));
            mbar_wait(&empty[sl], ((use >> sl) & 1) ^ 1);
          }
        }
        sl = __shfl_sync(0xffffffffu, sl, 0);
        if (hot) {
          if (lane == jj) {
            SingleQEntry e;
            e.dc = cur;
            e.slot = 0;
            e.fpar = 0;
            e.pad[0] = e.pad[1] = 0;
            queue[qi] = e;
            mbar_arrive(&qfull[qi]);
          }
          __syncwarp();
          continue;
        }
        const uint32_t fpar = (use >> sl) & 1u;
        use ^= 1u << sl;
        if (lane == jj) {
          SingleQEntry e;
          e.dc = cur;
          e.slot = static_cast<uint32_t>(sl);
          e.fpar = fpar;
          e.pad[0] = e.pad[1] = 0;
          queue[qi] = e;
          mbar_arrive(&qfull[qi]);
          mbar_expect_tx(&full[sl], ROWB);
          unsigned char* dst = ring + sl * ROWB;
          const size_t lz = static_cast<size_t>(cur.l);
          bulk_g2s(dst, Wb + lz * RG::WB, RG::WB, &full[sl]);
          if constexpr (ADAM) {
            bulk_g2s(dst + RG::WB, a.m + lz * d, RG::MB, &full[sl]);
            bulk_g2s(dst + RG::WB + RG::MB, a.v + lz * d, RG::MB, &full[sl]);
          }
        }
        __syncwarp();
      }
      cur = nxt;
      q1 = q2;
      q2 = q3;
    }
    return;
  }
  float wmax = 0.0f;
  // fp64 loss terms, evaluated lane-parallel 32 slots at a time (lane c holds
  // the c-th pending slot) and stored per slot for single_row_finalize
  int32_t pend_slot = 0;
  float pend_sc = 0.0f, pend_pt = 0.0f, pend_wn = 0.0f;
  int c_pend = 0;
  auto pend_loss = [&](int32_t slot, float sc, float pt, float wn) {
    if (lane == c_pend) {
      pend_slot = slot;
      pend_sc = sc;
      pend_pt = pt;
      pend_wn = wn;
    }
    if (++c_pend == 32) {
      A.slot_loss[pend_slot] = slot_loss(pend_sc, pend_pt, pend_wn);
      c_pend = 0;
    }
  };
  if (warp < n_mine) {  // the first label's embedding row towards L1
    mbar_wait(&qfull[warp % Q], (warp / Q) & 1);
    prefetch_emb_l1<NV>(fa.emb, queue[warp % Q].dc.slot0 / S, lane);
  }
  for (int i = warp; i < n_mine; i += kTmaConsumers) {
    const int qi = i % Q;
    mbar_wait(&qfull[qi], (i / Q) & 1);
    const SingleDesc dc = queue[qi].dc;
    const int r = static_cast<int>(queue[qi].slot);
    const uint32_t fpar = queue[qi].fpar;
    __syncwarp();
    if (lane == 0) mbar_arrive(&qempty[qi]);
    if (is_hot(dc.n)) continue;  // hot_label_kernel's
    // the first occurrence's embedding row (prefetched into L1 one label ago)
    float4 e0[NV];
    load_emb_row<NV>(fa.emb, dc.slot0 / S, lane, e0);
    {  // the next label's row towards L1, if its descriptor is already there
      const int in = i + kTmaConsumers;
      if (in < n_mine && mbar_test(&qfull[in % Q], (in / Q) & 1))
        prefetch_emb_l1<NV>(fa.emb, queue[in % Q].dc.slot0 / S, lane);
    }
    mbar_wait(&full[r], fpar);
    const unsigned char* ent = ring + r * ROWB;
    float4 p[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      if constexpr (BF16) {
        const uint2 u = *reinterpret_cast<const uint2*>(ent + (q * 128 + lane * 4) * 2);
        p[q] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                           __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
      } else {
        p[q] = *reinterpret_cast<const float4*>(ent + (q * 128 + lane * 4) * 4);
      }
    }
    constexpr bool EARLY = ADAM && ASTRA_SINGLE_ADAM_EARLY;
    float4 mr[EARLY ? NV : 1], vr[EARLY ? NV : 1];
    if constexpr (EARLY) {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        mr[q] = *reinterpret_cast<const float4*>(ent + RG::WB + (q * 128 + lane * 4) * 4);
        vr[q] = *reinterpret_cast<const float4*>(ent + RG::WB + RG::MB + (q * 128 + lane * 4) * 4);
      }
      regs_landed(mr);
      regs_landed(vr);
      regs_landed(p);
      __syncwarp();
      if (lane == 0) release(r);
    }
    const uint32_t n = dc.n;
    const size_t row = static_cast<size_t>(dc.l) * d;
    // the row update, element by element, from the label's gradient G(q)
    auto update_row = [&](auto G) {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const float4 gq = G(q);
        float4 np;
        const size_t el = row + q * 128 + lane * 4;
        if constexpr (ADAM) {
          float4 m4, v4;
          if constexpr (EARLY) {
            m4 = mr[q];
            v4 = vr[q];
          } else {
            m4 = *reinterpret_cast<const float4*>(ent + RG::WB + (q * 128 + lane * 4) * 4);
            v4 = *reinterpret_cast<const float4*>(ent + RG::WB + RG::MB + (q * 128 + lane * 4) * 4);
          }
          np.x = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p[q].x, gq.x, &m4.x, &v4.x);
          np.y = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p[q].y, gq.y, &m4.y, &v4.y);
          np.z = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p[q].z, gq.z, &m4.z, &v4.z);
          np.w = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p[q].w, gq.w, &m4.w, &v4.w);
          *reinterpret_cast<float4*>(a.m + el) = m4;
          *reinterpret_cast<float4*>(a.v + el) = v4;
        } else {
          np.x = upd_elem<false>(a, p[q].x, gq.x, nullptr, nullptr);
          np.y = upd_elem<false>(a, p[q].y, gq.y, nullptr, nullptr);
          np.z = upd_elem<false>(a, p[q].z, gq.z, nullptr, nullptr);
          np.w = upd_elem<false>(a, p[q].w, gq.w, nullptr, nullptr);
        }
        if constexpr (BF16) {
          uint2 o;
          o.x = static_cast<uint32_t>(f32_to_bf16_bits(np.x)) | (static_cast<uint32_t>(f32_to_bf16_bits(np.y)) << 16);
          o.y = static_cast<uint32_t>(f32_to_bf16_bits(np.z)) | (static_cast<uint32_t>(f32_to_bf16_bits(np.w)) << 16);
          *reinterpret_cast<uint2*>(static_cast<uint16_t*>(a.W) + el) = o;
        } else {
          *reinterpret_cast<float4*>(static_cast<float*>(a.W) + el) = np;
        }
        wmax = fmaxf(wmax, absmax4(np));
      }
    };
    auto grad_emb_add = [&](int b, float f) {
#ifdef ASTRA_SINGLE_DEBUG_NO_RED
      return;  // (experiment: measure the pass without the grad_emb reductions)
#endif
      if (f != 0.0f) {  // warp-uniform; dead slots (f = 0) add nothing to grad_emb
        float* ge = fa.grad_emb + static_cast<size_t>(b) * d + lane * 4;
#pragma unroll
        for (int q = 0; q < NV; ++q)
          red_add_v4(ge + q * 128, make_float4(__fmul_rn(f, p[q].x), __fmul_rn(f, p[q].y), __fmul_rn(f, p[q].z),
                                               __fmul_rn(f, p[q].w)));
      }
    };
    if (n == 1) {
      // ---- one occurrence (most labels): score, factor, grad_emb, then the
      // update straight from f * emb (0 + x = x, up to the sign of a zero)
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        acc = fmaf(p[q].x, e0[q].x, acc);
        acc = fmaf(p[q].y, e0[q].y, acc);
        acc = fmaf(p[q].z, e0[q].z, acc);
        acc = fmaf(p[q].w, e0[q].w, acc);
      }
      acc = warp_sum(acc);
      SlotMeta m;
      m.o = static_cast<int8_t>(dc.o0);
      m.yf = dc.yf0;
      m.w = dc.w0;
      float pt, wn;
      const float f = slot_factor_meta(m, acc, &pt, &wn);
      if (lane == 0) fa.factors[dc.slot0] = f;
      pend_loss(dc.slot0, acc, pt, wn);
      grad_emb_add(dc.slot0 / S, f);
      if constexpr (!ADAM) {  // W row consumed (Adam: after the moments, below)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) release(r);
      }
      update_row([&](int q) {
        return make_float4(__fmul_rn(f, e0[q].x), __fmul_rn(f, e0[q].y), __fmul_rn(f, e0[q].z), __fmul_rn(f, e0[q].w));
      });
    } else {
      // ---- several occurrences: in ascending b*S+s order (the two-kernel
      // update's summation order), the gradient accumulated in this warp's
      // shared scratch (lane-owned elements, no synchronisation)
      float* gs = gs_all + warp * d + lane * 4;
      const int32_t reg = sort_segment(a, dc.start, n, lane);
      const bool small = n <= 32;
      SlotMeta my;
      my.o = static_cast<int8_t>(dc.o0);
      my.yf = dc.yf0;
      my.w = dc.w0;
      if (small && lane < static_cast<int>(n) && reg != dc.slot0) my = slot_meta(fa, reg / S, reg - (reg / S) * S);
      // (prefetching the next occurrences' embedding rows into L1 was measured
      // slower: 0.665-0.675 vs 0.611 ms per C4 minibatch, profiles/r02/ab_lookahead.txt)
      for (uint32_t j = 0; j < n; ++j) {
        const int32_t slot = seg_slot(a, dc.start, n, reg, j);
        const int b = slot / S, s = slot - b * S;
        float4 e[NV];
        load_emb_row<NV>(fa.emb, b, lane, e);
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          acc = fmaf(p[q].x, e[q].x, acc);
          acc = fmaf(p[q].y, e[q].y, acc);
          acc = fmaf(p[q].z, e[q].z, acc);
          acc = fmaf(p[q].w, e[q].w, acc);
        }
        acc = warp_sum(acc);
        SlotMeta m;
        if (small) {
          m.o = static_cast<int8_t>(__shfl_sync(0xffffffffu, static_cast<int>(my.o), static_cast<int>(j)));
          m.yf = __shfl_sync(0xffffffffu, my.yf, static_cast<int>(j));
          m.w = __shfl_sync(0xffffffffu, my.w, static_cast<int>(j));
        } else {
          m = slot_meta(fa, b, s);
        }
        float pt, wn;
        const float f = slot_factor_meta(m, acc, &pt, &wn);
        if (lane == 0) fa.factors[slot] = f;
        pend_loss(slot, acc, pt, wn);
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          float4 gq = make_float4(__fmul_rn(f, e[q].x), __fmul_rn(f, e[q].y), __fmul_rn(f, e[q].z), __fmul_rn(f, e[q].w));
          if (j > 0) {
            const float4 o = *reinterpret_cast<const float4*>(gs + q * 128);
            gq = make_float4(__fadd_rn(o.x, gq.x), __fadd_rn(o.y, gq.y), __fadd_rn(o.z, gq.z), __fadd_rn(o.w, gq.w));
          }
          *reinterpret_cast<float4*>(gs + q * 128) = gq;
        }
        grad_emb_add(b, f);
      }
      if constexpr (!ADAM) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) release(r);
      }
      update_row([&](int q) { return *reinterpret_cast<const float4*>(gs + q * 128); });
    }
    if constexpr (ADAM && !EARLY) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) release(r);
    }
  }
  if (lane < c_pend) A.slot_loss[pend_slot] = slot_loss(pend_sc, pend_pt, pend_wn);
  push_wmax(a, wmax, lane);
}

// Per-row tail of the single pass (a CTA per batch row): the row's fp64 loss
// from the stored per-slot terms of its owned slots (thread-strided, then a
// fixed-order reduction: deterministic), the keep scale and finiteness check
// of grad_emb. bound_rows = 0: finiteness was proven up front. d % 128 == 0.
constexpr int kRowFinThreads = 256;
__global__ void __launch_bounds__(kRowFinThreads) single_row_finalize(FwdArgs a, const double* slot_loss,
                                                                      const int32_t* mode) {
  pdl_entry();
  if (!*mode) return;
  __shared__ double sl[kRowFinThreads / 32];
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double l = 0.0;
  for (int s = threadIdx.x; s < a.S; s += kRowFinThreads) {
    const size_t slot = static_cast<size_t>(b) * a.S + s;
    const int64_t loc = static_cast<int64_t>(a.ids[slot]) - a.off;
    if (loc >= 0 && loc < a.Lloc) l += slot_loss[slot];
  }
  l = warp_sum(l);
  if (lane == 0) sl[warp] = l;
  bool bad = false;
  float* ge = a.grad_emb + static_cast<size_t>(b) * a.d;
  const float* kp = a.keep ? a.keep + static_cast<size_t>(b) * a.d : nullptr;
  for (int k = threadIdx.x * 4; k < a.d; k += kRowFinThreads * 4) {
    float4 g = *reinterpret_cast<const float4*>(ge + k);
    if (kp) {
      const float4 kk = *reinterpret_cast<const float4*>(kp + k);
      g = make_float4(__fmul_rn(g.x, kk.x), __fmul_rn(g.y, kk.y), __fmul_rn(g.z, kk.z), __fmul_rn(g.w, kk.w));
      *reinterpret_cast<float4*>(ge + k) = g;
    }
    bad |= !(isfinite(g.x) && isfinite(g.y) && isfinite(g.z) && isfinite(g.w));
  }
  if (bad) a.status[ASTRA_STATUS_NONFINITE_GRAD_EMB] = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRowFinThreads / 32; ++w) t += sl[w];
    a.loss_rows[b] = t;
    a.bound_rows[b] = 0.0;
  }
}

// The hot labels of the single pass (is_hot): CTA per label (grid-stride over
// the device-side list). Phase A, warps over the label's occurrences in any
// order: score (the pass's lane layout, fma order and butterfly: the same
// bits), factor, fp64 loss term, grad_emb[b] += f * W_old (vector
// reductions) — independent per occurrence, so a label with hundreds of
// occurrences costs a few rounds of 8 warps instead of a serial walk. Phase B:
// the occurrences sorted ascending in shared memory, each thread sums its 4
// elements' gradient in that order (the two-kernel update's order and
// roundings: W' stays bit-identical), then the SGD / Adam row update.
constexpr int kHotThreads = 256;
template <int NV, bool BF16, bool ADAM>
__global__ void __launch_bounds__(kHotThreads) hot_label_kernel(SingleArgs A, const int32_t* hot_u,
                                                                 const uint32_t* n_hot, int sort_cap) {
  pdl_entry();
  constexpr int d = NV * 128;
  if (!*A.mode) return;
  const UpdArgs& a = A.u;
  const FwdArgs& fa = A.f;
  const int S = fa.S;
  extern __shared__ int32_t hot_sorted[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kWarps = kHotThreads / 32;
  float wmax = 0.0f;
  const uint32_t nh = *n_hot;
  for (uint32_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const uint32_t u = static_cast<uint32_t>(hot_u[h]);
    const int32_t l = a.uniq[u];
    const uint32_t start = A.ustart[u], n = A.ucnt[u];
    const size_t row = static_cast<size_t>(l) * d;
    // ---- phase A
    float4 p[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) p[q] = load_w4<BF16>(a.W, row + q * 128 + lane * 4);
    for (uint32_t j = warp; j < n; j += kWarps) {
      const int32_t slot = a.perm[start + j];
      const int b = slot / S, s = slot - b * S;
      float4 e[NV];
      load_emb_row<NV>(fa.emb, b, lane, e);
      const SlotMeta m = slot_meta(fa, b, s);
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        acc = fmaf(p[q].x, e[q].x, acc);
        acc = fmaf(p[q].y, e[q].y, acc);
        acc = fmaf(p[q].z, e[q].z, acc);
        acc = fmaf(p[q].w, e[q].w, acc);
      }
      acc = warp_sum(acc);
      float pt, wn;
      const float f = slot_factor_meta(m, acc, &pt, &wn);
      if (lane == 0) {
        fa.factors[slot] = f;
        A.slot_loss[slot] = slot_loss(acc, pt, wn);
      }
      if (f != 0.0f) {
        float* ge = fa.grad_emb + static_cast<size_t>(b) * d + lane * 4;
#pragma unroll
        for (int q = 0; q < NV; ++q)
          red_add_v4(ge + q * 128, make_float4(__fmul_rn(f, p[q].x), __fmul_rn(f, p[q].y), __fmul_rn(f, p[q].z),
                                               __fmul_rn(f, p[q].w)));
      }
    }
    // ---- phase B: ascending slot order (bitonic sort of the padded segment)
    int P2 = 1;
    while (P2 < static_cast<int>(n)) P2 <<= 1;
    for (int i = threadIdx.x; i < P2; i += kHotThreads)
      hot_sorted[i] = i < static_cast<int>(n) ? a.perm[start + i] : INT_MAX;
    __syncthreads();  // (also: the factors written in phase A are visible to the block)
    for (int size = 2; size <= P2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < P2; i += kHotThreads) {
          const int jx = i ^ stride;
          if (jx > i) {
            const bool up = (i & size) == 0;
            const int32_t x = hot_sorted[i], y = hot_sorted[jx];
            if ((x > y) == up) {
              hot_sorted[i] = y;
              hot_sorted[jx] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    if (threadIdx.x < d / 4) {
      const int t4 = threadIdx.x * 4;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
      for (uint32_t j = 0; j < n; ++j) {
        const int32_t slot = hot_sorted[j];
        const float f = fa.factors[slot];
        const float4 x = *reinterpret_cast<const float4*>(fa.emb + static_cast<size_t>(slot / S) * d + t4);
        const float4 fx = make_float4(__fmul_rn(f, x.x), __fmul_rn(f, x.y), __fmul_rn(f, x.z), __fmul_rn(f, x.w));
        g = j == 0 ? fx : make_float4(__fadd_rn(g.x, fx.x), __fadd_rn(g.y, fx.y), __fadd_rn(g.z, fx.z), __fadd_rn(g.w, fx.w));
      }
      const size_t el = row + t4;
      const float4 p4 = load_w4<BF16>(a.W, el);
      float4 np;
      if constexpr (ADAM) {
        float4 m4 = *reinterpret_cast<const float4*>(a.m + el), v4 = *reinterpret_cast<const float4*>(a.v + el);
        np.x = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p4.x, g.x, &m4.x, &v4.x);
        np.y = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p4.y, g.y, &m4.y, &v4.y);
        np.z = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p4.z, g.z, &m4.z, &v4.z);
        np.w = upd_elem<true, BF16 && ASTRA_ADAM_FAST>(a, p4.w, g.w, &m4.w, &v4.w);
        *reinterpret_cast<float4*>(a.m + el) = m4;
        *reinterpret_cast<float4*>(a.v + el) = v4;
      } else {
        np.x = upd_elem<false>(a, p4.x, g.x, nullptr, nullptr);
        np.y = upd_elem<false>(a, p4.y, g.y, nullptr, nullptr);
        np.z = upd_elem<false>(a, p4.z, g.z, nullptr, nullptr);
        np.w = upd_elem<false>(a, p4.w, g.w, nullptr, nullptr);
      }
      if constexpr (BF16) {
        uint2 o;
        o.x = static_cast<uint32_t>(f32_to_bf16_bits(np.x)) | (static_cast<uint32_t>(f32_to_bf16_bits(np.y)) << 16);
        o.y = static_cast<uint32_t>(f32_to_bf16_bits(np.z)) | (static_cast<uint32_t>(f32_to_bf16_bits(np.w)) << 16);
        *reinterpret_cast<uint2*>(static_cast<uint16_t*>(a.W) + el) = o;
      } else {
        *reinterpret_cast<float4*>(static_cast<float*>(a.W) + el) = np;
      }
      wmax = fmaxf(wmax, absmax4(np));
    }
    __syncthreads();  // before the next label reuses the sort buffer
  }
  push_wmax(a, wmax, lane);
}

// The chain's first kernel: zeroes the label counts, the single pass's bounds
// block and the status words (one launch instead of three memsets).
__global__ void __launch_bounds__(256) step_zero_kernel(uint32_t* counts, int64_t Lloc, unsigned* bar,
                                                        int32_t* status) {
  pdl_entry();
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n4 = Lloc / 4;  // (workspace arrays are 256-byte aligned)
  for (int64_t i = t; i < n4; i += nt) reinterpret_cast<uint4*>(counts)[i] = make_uint4(0u, 0u, 0u, 0u);
  for (int64_t i = n4 * 4 + t; i < Lloc; i += nt) counts[i] = 0u;
  if (bar && t < 8) bar[t] = 0u;
  if (t < ASTRA_STATUS_WORDS) status[t] = 0;
}

template <int NV, bool BF16, bool ADAM>
void launch_hot_nv(const SingleArgs& A, const int32_t* hot_u, const uint32_t* n_hot, int sort_cap, cudaStream_t st) {
  const size_t smem = sizeof(int32_t) * static_cast<size_t>(sort_cap);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(hot_label_kernel<NV, BF16, ADAM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(int32_t) * kHotMax));
    attr = true;
  }
  launch_pdl(hot_label_kernel<NV, BF16, ADAM>, 2 * num_sms(), kHotThreads, smem, st, A, hot_u, n_hot, sort_cap);
}

template <int NV, bool BF16, bool ADAM>
void launch_single_tma(const SingleArgs& A, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(step_single_tma<NV, BF16, ADAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  using RG = SingleRing<NV, BF16, ADAM>;
  launch_pdl(step_single_tma<NV, BF16, ADAM>, RG::CTAS * num_sms(), kTmaThreads, RG::smem(), st, A);
}

template <bool BF16, bool ADAM>
void launch_single_nv(int nv, const SingleArgs& A, cudaStream_t st) {
  switch (nv) {
    case 1: launch_single_tma<1, BF16, ADAM>(A, st); break;
    case 2: launch_single_tma<2, BF16, ADAM>(A, st); break;
    case 4: launch_single_tma<4, BF16, ADAM>(A, st); break;
    case 6: launch_single_tma<6, BF16, ADAM>(A, st); break;
  }
}

// apply_classifier_updates_arrays: explicit (ids, grads) form.
__global__ void apply_check_kernel(const float* grads, int64_t n, int32_t* status) {
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= !isfinite(grads[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) status[ASTRA_STATUS_NONFINITE_GRAD] = 1;
}

template <bool BF16>
__global__ void apply_rows_kernel(void* W, int d, const int64_t* ids, const float* grads, int64_t U, float lr,
                                  float wd, const int32_t* status) {
  if (status[ASTRA_STATUS_NONFINITE_GRAD]) return;
  const int64_t n = U * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / d, k = i - r * d;
    const size_t el = static_cast<size_t>(ids[r]) * d + k;
    float p = load_p<BF16>(W, el);
    store_p<BF16>(W, el, __fsub_rn(p, __fmul_rn(lr, __fadd_rn(grads[i], __fmul_rn(wd, p)))));
  }
}

template <int NV, bool BF16>
bool launch_forward_vec(const FwdArgs& a, cudaStream_t st) {
  const size_t smem = tma_fwd_smem<NV, BF16>(a.S);
  if (smem > 200 * 1024) return false;  // (S > ~20K slots: the generic kernel)
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(slot_forward_tma<NV, BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  launch_pdl(slot_forward_tma<NV, BF16>, a.B, kTmaThreads, smem, st, a);
  return true;
}

template <int NV, bool BF16, bool ADAM>
void launch_upd_tma(const UpdArgs& a, int grid, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(label_update_tma<NV, BF16, ADAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  launch_pdl(label_update_tma<NV, BF16, ADAM>, grid, kTmaThreads, smem, st, a);
}

template <bool BF16, bool ADAM>
int launch_update(const UpdArgs& a, int max_ctas, cudaStream_t st) {
  const int nv = a.d % 128 == 0 ? a.d / 128 : 0;
  // (the check pass returns at once unless the bound tripped: a small grid keeps that cheap)
  launch_pdl(label_update_kernel<BF16, ADAM, true>, std::min(max_ctas, 2 * num_sms()), kUpdThreads, 0, st, a);
  ASTRA_LAUNCHED("label_check");
  if (nv == 1 || nv == 2 || nv == 4 || nv == 6 || nv == 8) {
    const int grid = (ADAM && nv > 6 ? 2 : (ADAM ? ASTRA_UPD_ADAM_CTAS : 3)) * num_sms();  // = upd_tma_ctas<nv, ADAM>()
    size_t smem = 0;
    switch (nv) {
      case 1: smem = UpdRing<1, BF16, ADAM>::smem(); break;
      case 2: smem = UpdRing<2, BF16, ADAM>::smem(); break;
      case 4: smem = UpdRing<4, BF16, ADAM>::smem(); break;
      case 6: smem = UpdRing<6, BF16, ADAM>::smem(); break;
      case 8: smem = UpdRing<8, BF16, ADAM>::smem(); break;
    }
    switch (nv) {
      case 1: launch_upd_tma<1, BF16, ADAM>(a, grid, smem, st); break;
      case 2: launch_upd_tma<2, BF16, ADAM>(a, grid, smem, st); break;
      case 4: launch_upd_tma<4, BF16, ADAM>(a, grid, smem, st); break;
      case 6: launch_upd_tma<6, BF16, ADAM>(a, grid, smem, st); break;
      case 8: launch_upd_tma<8, BF16, ADAM>(a, grid, smem, st); break;
    }
    ASTRA_LAUNCHED("label_update_tma");
    return ASTRA_OK;
  }
  launch_pdl(label_update_kernel<BF16, ADAM, false>, max_ctas, kUpdThreads, 0, st, a);
  ASTRA_LAUNCHED("label_update");
  return ASTRA_OK;
}

struct StepWs {
  unsigned* bar;
  double* sf_acc;
  unsigned* emax_acc;
  float* factors;
  int32_t* rank;
  int32_t* perm;
  int32_t* perm2;
  uint32_t* counts;
  uint32_t* offsets;
  int32_t* uniq;
  uint32_t* blk_slots;
  uint32_t* blk_nz;
  uint32_t* U;
  double* loss_rows;
  double* bound_rows;
  int32_t* mode;
  double* slot_loss;
  uint32_t* ustart;
  uint32_t* ucnt;
  uint32_t* n_hot;  // (in the memset bounds block)
  int32_t* hot_u;   // hot labels' positions in uniq
};

size_t carve_step(void* base, size_t cap, int B, int S, int64_t Lloc, StepWs* w) {
  Carve c(base, cap);
  const int64_t n = static_cast<int64_t>(B) * S;
  const int64_t nb = (Lloc + kScanTile - 1) / kScanTile;
  w->factors = c.take<float>(n);
  w->rank = c.take<int32_t>(n);
  w->perm = c.take<int32_t>(n);
  w->perm2 = c.take<int32_t>(n);
  w->counts = c.take<uint32_t>(Lloc);
  w->offsets = c.take<uint32_t>(Lloc);
  w->uniq = c.take<int32_t>(n < Lloc ? n : Lloc);
  w->blk_slots = c.take<uint32_t>(nb);
  w->blk_nz = c.take<uint32_t>(nb);
  w->U = c.take<uint32_t>(1);
  w->loss_rows = c.take<double>(B);
  w->bound_rows = c.take<double>(B);
  // one 32-byte block (a single memset): bar, emax_acc, (pad x2), the fp64 accumulator
  w->bar = c.take<unsigned>(8);
  w->emax_acc = w->bar ? w->bar + 1 : nullptr;
  w->sf_acc = w->bar ? reinterpret_cast<double*>(w->bar + 4) : nullptr;
  w->mode = c.take<int32_t>(4);
  w->slot_loss = c.take<double>(n);
  w->ustart = c.take<uint32_t>(n < Lloc ? n : Lloc);
  w->ucnt = c.take<uint32_t>(n < Lloc ? n : Lloc);
  w->n_hot = w->bar ? w->bar + 2 : nullptr;
  w->hot_u = c.take<int32_t>(n / (kHotOcc + 1) + 1);
  return c.off;
}

}  // namespace

std::atomic<int> g_step_deterministic{0};

void set_step_deterministic(int on) { g_step_deterministic.store(on ? 1 : 0); }

size_t step_workspace_size(int B, int S, int d, int64_t Lloc) {
  (void)d;
  StepWs w;
  return carve_step(nullptr, 0, B, S, Lloc, &w);
}

int slate_step(const float* emb, const float* keep, const int32_t* ids, const int8_t* y, const int8_t* origin,
               int64_t origin_stride, const float* weights, int64_t weights_stride, const float* factors_in, int B,
               int S, int d, void* W, int w_dtype, float* adam_m, float* adam_v, int optimizer, int64_t Lloc,
               int64_t off, double lr, double wd, double b1, double b2, double eps, int64_t adam_step, float* grad_emb,
               double* loss_out, int32_t* status, float* factors_out, float* w_absmax, void* workspace,
               size_t ws_bytes, cudaStream_t st) {
  if (B < 0 || S < 0 || d <= 0 || Lloc < 0) return set_error(ASTRA_ERR_CONFIG, "slate_step: bad shape");
  if (Lloc >= (int64_t(1) << 31) || static_cast<int64_t>(B) * S >= (int64_t(1) << 31))
    return set_error(ASTRA_ERR_CONFIG, "slate_step: shard too large for 32-bit slot indices");
  if (w_dtype != ASTRA_W_FP32 && w_dtype != ASTRA_W_BF16) return set_error(ASTRA_ERR_CONFIG, "bad w_dtype");
  if (optimizer == ASTRA_OPT_ADAM && (!adam_m || !adam_v))
    return set_error(ASTRA_ERR_CONFIG, "Adam needs moment buffers");
  StepWs w;
  size_t need = carve_step(workspace, ws_bytes, B, S, Lloc, &w);
  if (!workspace || ws_bytes < need) return set_error(ASTRA_ERR_CONFIG, "step workspace too small (%zu < %zu)", ws_bytes, need);
  if (B == 0 || S == 0 || Lloc == 0) {
    ASTRA_TRY(check_cuda(cudaMemsetAsync(status, 0, sizeof(int32_t) * ASTRA_STATUS_WORDS, st), "memset status"));
  }
  if (B == 0 || S == 0) {  // (otherwise finalize_kernel assigns the loss)
    ASTRA_TRY(check_cuda(cudaMemsetAsync(loss_out, 0, sizeof(double), st), "memset loss"));
    if (B) ASTRA_TRY(check_cuda(cudaMemsetAsync(grad_emb, 0, sizeof(float) * B * d, st), "memset grad_emb"));
    return ASTRA_OK;
  }
  const bool bf16 = w_dtype == ASTRA_W_BF16;
  FwdArgs fa;
  fa.emb = emb;
  fa.keep = keep;
  fa.ids = ids;
  fa.y = y;
  fa.origin = origin;
  fa.origin_stride = origin_stride;
  fa.weights = weights;
  fa.weights_stride = weights_stride;
  fa.factors_in = factors_in;
  fa.B = B;
  fa.S = S;
  fa.d = d;
  fa.W = W;
  fa.Lloc = Lloc;
  fa.off = off;
  fa.grad_emb = grad_emb;
  fa.factors = factors_out ? factors_out : w.factors;
  fa.loss_rows = w.loss_rows;
  fa.bound_rows = w.bound_rows;
  fa.status = status;
  const int nv = d % 128 == 0 ? d / 128 : 0;
  const bool aligned = (reinterpret_cast<uintptr_t>(emb) % 16 == 0) && (reinterpret_cast<uintptr_t>(W) % 16 == 0);
  const bool adam = optimizer == ASTRA_OPT_ADAM;
  const bool chunkable = !factors_in && aligned && Lloc > 0 && (nv == 1 || nv == 2 || nv == 4 || nv == 6 || nv == 8);
  static const bool single_env = [] {
    // ASTRA_STEP_SINGLE=0: the deterministic two-kernel schedule (gather forward,
    // then label-major update) instead of the single label-major pass
    const char* e = getenv("ASTRA_STEP_SINGLE");
    return e ? atoi(e) != 0 : true;
  }();
  // Adam: with the MUFU sqrt / reciprocal update on bf16 W the single pass
  // measures slightly faster than the two-kernel schedule at the C5 shard
  // (15M labels, 4096 x 2344 slates, under the refresh's power cap: step 4.21
  // vs 4.35 ms, profiles/r02s3/ab_adam_single_c5.txt); with the IEEE sequences
  // it was slower (6.78 vs 5.65 ms). ASTRA_STEP_SINGLE_ADAM=0 selects the
  // two-kernel schedule (parity-tested bit-identical). nv = 8 spills.
  static const bool single_adam = [] {
    const char* e = getenv("ASTRA_STEP_SINGLE_ADAM");
    return e == nullptr || atoi(e) != 0;
  }();
  const bool single = single_env && !g_step_deterministic.load() && chunkable && nv <= 6 &&
                      (!adam || single_adam) &&
                      reinterpret_cast<uintptr_t>(grad_emb) % 16 == 0;  // (vector reductions into it)
  if (single) fa.skip = w.mode;

  // counting sort of the slots by local label id (+ the single pass's bounds and decision)
  const int64_t n = static_cast<int64_t>(B) * S;
  const int64_t nb = (Lloc + kScanTile - 1) / kScanTile;
  if (nb > 1024 * 1024) return set_error(ASTRA_ERR_CONFIG, "label shard too large");
  const int sms = num_sms();
  const int grid_n = static_cast<int>(std::min<int64_t>((n + 255) / 256, 8LL * sms));
  if (Lloc > 0) {
    launch_pdl(step_zero_kernel, static_cast<int>(std::min<int64_t>((Lloc / 4 + 255) / 256 + 1, 4LL * sms)), 256, 0,
               st, w.counts, Lloc, single ? w.bar : nullptr, status);
    ASTRA_LAUNCHED("step_zero");
    // (single pass: count_kernel also zeroes grad_emb, which the pass reduces into)
    launch_pdl(count_kernel, grid_n, 256, 0, st, ids, n, off, Lloc, w.counts, w.rank, status, weights, weights_stride,
               S, emb, static_cast<int64_t>(B) * d, single ? w.sf_acc : nullptr, w.emax_acc,
               single ? grad_emb : nullptr);
    ASTRA_LAUNCHED("count");
    launch_pdl(scan_reduce_kernel, static_cast<int>(nb), kScanThreads, 0, st, w.counts, Lloc, w.blk_slots, w.blk_nz);
    ASTRA_LAUNCHED("scan_reduce");
    launch_pdl(scan_top_kernel, 1, 1024, 0, st, w.blk_slots, w.blk_nz, static_cast<int>(nb), w.U, w.sf_acc,
               w.emax_acc, w_absmax, single ? w.mode : nullptr, d);
    ASTRA_LAUNCHED("scan_top");
    launch_pdl(scan_apply_kernel, static_cast<int>(nb), kScanThreads, 0, st, w.counts, Lloc, w.blk_slots, w.blk_nz,
               w.offsets, w.uniq, single ? w.ustart : nullptr, w.ucnt, single ? w.n_hot : nullptr,
               single ? w.hot_u : nullptr);
    ASTRA_LAUNCHED("scan_apply");
    launch_pdl(scatter_kernel, grid_n, 256, 0, st, ids, w.rank, n, off, w.offsets, w.perm);
    ASTRA_LAUNCHED("scatter");
  }

  UpdArgs ua;
  ua.emb = emb;
  ua.factors = fa.factors;
  ua.uniq = w.uniq;
  ua.U = w.U;
  ua.offsets = w.offsets;
  ua.counts = w.counts;
  ua.perm = w.perm;
  ua.perm2 = w.perm2;
  ua.S = S;
  ua.d = d;
  ua.W = W;
  ua.m = adam_m;
  ua.v = adam_v;
  ua.lr = static_cast<float>(lr);  // np.float32(lr), classifiers.py:82
  ua.wd = static_cast<float>(wd);
  ua.status = status;
  ua.c1 = ua.c2 = ua.eps = ua.neg_step = 0.0f;
  if (optimizer == ASTRA_OPT_ADAM) {
    // torch.optim.SparseAdam: scalars in double, rounded to fp32 when applied
    double bc1 = 1.0 - pow(b1, static_cast<double>(adam_step));
    double bc2 = 1.0 - pow(b2, static_cast<double>(adam_step));
    ua.c1 = static_cast<float>(1.0 - b1);
    ua.c2 = static_cast<float>(1.0 - b2);
    ua.eps = static_cast<float>(eps);
    ua.neg_step = static_cast<float>(-(lr * sqrt(bc2) / bc1));
  }
  ua.w_absmax = w_absmax;
  ua.skip = single ? w.mode : nullptr;
  if (single) {
    SingleArgs SA;
    SA.f = fa;
    SA.u = ua;
    SA.slot_loss = w.slot_loss;
    SA.mode = w.mode;
    SA.ustart = w.ustart;
    SA.ucnt = w.ucnt;
    {
      // the hot labels first (the pass skips them; disjoint rows, additive grad_emb)
      int sort_cap = 1;
      while (sort_cap < static_cast<int>(std::min<int64_t>(n, kHotMax))) sort_cap <<= 1;
      auto hot = [&](auto bf_tag, auto adam_tag) {
        constexpr bool BF = decltype(bf_tag)::value, AD = decltype(adam_tag)::value;
        switch (nv) {
          case 1: launch_hot_nv<1, BF, AD>(SA, w.hot_u, w.n_hot, sort_cap, st); break;
          case 2: launch_hot_nv<2, BF, AD>(SA, w.hot_u, w.n_hot, sort_cap, st); break;
          case 4: launch_hot_nv<4, BF, AD>(SA, w.hot_u, w.n_hot, sort_cap, st); break;
          case 6: launch_hot_nv<6, BF, AD>(SA, w.hot_u, w.n_hot, sort_cap, st); break;
        }
      };
      using T = std::true_type;
      using F = std::false_type;
      if (bf16)
        adam ? hot(T(), T()) : hot(T(), F());
      else
        adam ? hot(F(), T()) : hot(F(), F());
      ASTRA_LAUNCHED("hot_label");
    }
    KernelTimer kt("step_single", st);
    if (bf16)
      adam ? launch_single_nv<true, true>(nv, SA, st) : launch_single_nv<true, false>(nv, SA, st);
    else
      adam ? launch_single_nv<false, true>(nv, SA, st) : launch_single_nv<false, false>(nv, SA, st);
    ASTRA_LAUNCHED("step_single");
  }
  {
    KernelTimer kt_fwd("slot_forward", st);
    bool launched = false;
    if (aligned && (nv == 1 || nv == 2 || nv == 4 || nv == 6 || nv == 8)) {
      switch (nv * 2 + (bf16 ? 1 : 0)) {
        case 2: launched = launch_forward_vec<1, false>(fa, st); break;
        case 3: launched = launch_forward_vec<1, true>(fa, st); break;
        case 4: launched = launch_forward_vec<2, false>(fa, st); break;
        case 5: launched = launch_forward_vec<2, true>(fa, st); break;
        case 8: launched = launch_forward_vec<4, false>(fa, st); break;
        case 9: launched = launch_forward_vec<4, true>(fa, st); break;
        case 12: launched = launch_forward_vec<6, false>(fa, st); break;
        case 13: launched = launch_forward_vec<6, true>(fa, st); break;
        case 16: launched = launch_forward_vec<8, false>(fa, st); break;
        case 17: launched = launch_forward_vec<8, true>(fa, st); break;
      }
    }
    if (!launched) {
      size_t smem = sizeof(float) * static_cast<size_t>(d) * (1 + kFwdWarps);
      if (smem > 200 * 1024) return set_error(ASTRA_ERR_CONFIG, "slate_step: d=%d too large", d);
      if (bf16) {
        cudaFuncSetAttribute(slot_forward_generic<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_pdl(slot_forward_generic<true>, B, kFwdThreads, smem, st, fa);
      } else {
        cudaFuncSetAttribute(slot_forward_generic<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_pdl(slot_forward_generic<false>, B, kFwdThreads, smem, st, fa);
      }
    }
    ASTRA_LAUNCHED("slot_forward");
  }
  if (single) {
    launch_pdl(single_row_finalize, B, kRowFinThreads, 0, st, fa, static_cast<const double*>(w.slot_loss),
               static_cast<const int32_t*>(w.mode));
    ASTRA_LAUNCHED("single_row_finalize");
  }
  launch_pdl(finalize_kernel, 1, 1024, 0, st, static_cast<const double*>(w.loss_rows),
             static_cast<const double*>(w.bound_rows), B, loss_out, status);
  ASTRA_LAUNCHED("finalize");

  if (Lloc == 0) return ASTRA_OK;
  const int upd_ctas = 16 * sms;
  KernelTimer kt_upd("label_update", st);
  if (optimizer == ASTRA_OPT_ADAM)
    return bf16 ? launch_update<true, true>(ua, upd_ctas, st) : launch_update<false, true>(ua, upd_ctas, st);
  return bf16 ? launch_update<true, false>(ua, upd_ctas, st) : launch_update<false, false>(ua, upd_ctas, st);
}

int apply_updates(void* W, int w_dtype, int64_t n_labels, int d, const int64_t* ids, const float* grads, int64_t U,
                  float lr, float wd, int32_t* status, cudaStream_t st) {
  (void)n_labels;
  ASTRA_TRY(check_cuda(cudaMemsetAsync(status, 0, sizeof(int32_t) * ASTRA_STATUS_WORDS, st), "memset status"));
  if (U == 0) return ASTRA_OK;
  const int64_t n = U * d;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 8LL * num_sms()));
  apply_check_kernel<<<grid, 256, 0, st>>>(grads, n, status);
  ASTRA_LAUNCHED("apply_check");
  if (w_dtype == ASTRA_W_BF16)
    apply_rows_kernel<true><<<grid, 256, 0, st>>>(W, d, ids, grads, U, lr, wd, status);
  else
    apply_rows_kernel<false><<<grid, 256, 0, st>>>(W, d, ids, grads, U, lr, wd, status);
  ASTRA_LAUNCHED("apply_rows");
  return ASTRA_OK;
}

}  // namespace astra
