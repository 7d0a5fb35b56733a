// dense.cu — the elementwise half of the all-negatives (full-loss) arm,
// train_full_loss_baseline (trainer.py:563-616), and of the dense probe loss
// _probe_full_loss (trainer.py:398-403). The three GEMMs of the arm
// (E W^T, G W, G^T E) are astra_gemm_f32 (dense_tc.cu, 3xTF32 tensor cores);
// the elementwise parts run here:
//   * dense_bce: over the B x L scores, G = f32(sigmoid(s)) - y with the
//     reference's float64 sigmoid 0.5 (1 + tanh(s / 2)) (loss.py:45-47) cast
//     to fp32 as trainer.py:597 does, and the float64 loss
//     sum y sp(-s) + (1 - y) sp(s) (trainer.py:595, loss.py:36-42), computed
//     as sum_all sp(s) - sum_pos s (sp(-s) - sp(s) = -s); the positives come
//     as a CSR (sorted, distinct ids per row) instead of the dense y matrix;
//     fixed-order reductions (deterministic);
//   * dense_sgd: W -= f32(lr) (g + f32(wd) W) over every row, each op rounded
//     like NumPy (trainer.py:604-606).
// Scores may be fp32 (the training step) or fp64 (the probe, which scores in
// float64, trainer.py:399-400).
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace astra {
namespace {

constexpr int kDenseThreads = 256;
constexpr int kDenseBlocksMax = 4096;


__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kDenseThreads / 32; ++w) t += sh[w];
  return t;  // valid in thread 0
}

template <typename T>
__global__ void __launch_bounds__(kDenseThreads) dense_bce_kernel(const T* S, int64_t n, float* G, double* part) {
  __shared__ double sh[kDenseThreads / 32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kDenseThreads) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * kDenseThreads) {
    const double s = static_cast<double>(S[i]);
    // one exp serves both: sp(s) = max(s, 0) + log1p(e) and, for s >= -15,
    // sigmoid = 1 / (1 + e) or e / (1 + e) with e = exp(-|s|) — the same value
    // to fp64 accuracy as the reference's 0.5 (1 + tanh(s / 2)), hence the
    // same fp32 after the cast; below -15 the reference's formula loses digits
    // to cancellation (1 + tanh ~ 2e), so that rare branch evaluates it as is
    const double e = exp(-fabs(s));
    if (G) {
      double sg;
      if (s >= -15.0)
        sg = s >= 0.0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
      else
        sg = 0.5 * (1.0 + tanh(0.5 * s));
      G[i] = static_cast<float>(sg);
    }
    acc += fmax(s, 0.0) + log1p(e);
  }
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// One CTA per row: the positives' correction -s to the loss, G -= 1.
template <typename T>
__global__ void __launch_bounds__(kDenseThreads) dense_pos_kernel(const T* S, int64_t L, const int64_t* indptr,
                                                                  const int32_t* ids, float* G, double* part) {
  __shared__ double sh[kDenseThreads / 32];
  const int b = blockIdx.x;
  double acc = 0.0;
  for (int64_t j = indptr[b] + threadIdx.x; j < indptr[b + 1]; j += kDenseThreads) {
    const int64_t el = static_cast<int64_t>(b) * L + ids[j];
    acc -= static_cast<double>(S[el]);
    if (G) G[el] = __fsub_rn(G[el], 1.0f);
  }
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) part[b] = t;
}

// One CTA: thread t sums parts t, t + 1024, ... of each list, then a fixed
// tree over the threads (deterministic; the single-thread loop over ~5K
// partials took 0.1 ms).
__global__ void __launch_bounds__(1024) dense_loss_finalize(const double* part, int n1, const double* part2, int n2,
                                                            double* out) {
  __shared__ double sh[1024];
  double t = 0.0, u = 0.0;
  for (int i = threadIdx.x; i < n1; i += 1024) t += part[i];
  for (int i = threadIdx.x; i < n2; i += 1024) u += part2[i];
  sh[threadIdx.x] = t + u;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void __launch_bounds__(kDenseThreads) dense_sgd_kernel(float* W, const float* g, int64_t n, float lr,
                                                                  float wd) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kDenseThreads) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * kDenseThreads) {
    const float p = W[i];
    W[i] = __fsub_rn(p, __fmul_rn(lr, __fadd_rn(g[i], __fmul_rn(wd, p))));
  }
}

int grid_for(int64_t n) {
  return static_cast<int>(std::min<int64_t>((n + kDenseThreads - 1) / kDenseThreads,
                                            std::min<int64_t>(kDenseBlocksMax, 16LL * num_sms())));
}

}  // namespace

size_t dense_workspace_size(int B) {
  return sizeof(double) * (static_cast<size_t>(kDenseBlocksMax) + static_cast<size_t>(B > 0 ? B : 0) + 64);
}

int dense_bce(const void* S, int s_f64, int B, int64_t L, const int64_t* pos_indptr, const int32_t* pos_ids,
              float* G, double* loss_out, void* workspace, size_t ws_bytes, cudaStream_t st) {
  if (B < 0 || L < 0) return set_error(ASTRA_ERR_CONFIG, "dense_bce: bad shape");
  if (!workspace || ws_bytes < dense_workspace_size(B))
    return set_error(ASTRA_ERR_CONFIG, "dense_bce: workspace too small");
  const int64_t n = static_cast<int64_t>(B) * L;
  if (n == 0) return check_cuda(cudaMemsetAsync(loss_out, 0, sizeof(double), st), "memset loss");
  double* part = static_cast<double*>(workspace);
  double* part2 = part + kDenseBlocksMax;
  const int grid = grid_for(n);
  if (s_f64) {
    dense_bce_kernel<double><<<grid, kDenseThreads, 0, st>>>(static_cast<const double*>(S), n, G, part);
    ASTRA_LAUNCHED("dense_bce");
    if (B) dense_pos_kernel<double><<<B, kDenseThreads, 0, st>>>(static_cast<const double*>(S), L, pos_indptr, pos_ids, G, part2);
  } else {
    dense_bce_kernel<float><<<grid, kDenseThreads, 0, st>>>(static_cast<const float*>(S), n, G, part);
    ASTRA_LAUNCHED("dense_bce");
    if (B) dense_pos_kernel<float><<<B, kDenseThreads, 0, st>>>(static_cast<const float*>(S), L, pos_indptr, pos_ids, G, part2);
  }
  ASTRA_LAUNCHED("dense_pos");
  dense_loss_finalize<<<1, 1024, 0, st>>>(part, grid, part2, B, loss_out);
  ASTRA_LAUNCHED("dense_loss_finalize");
  return ASTRA_OK;
}

int dense_sgd(float* W, const float* grads, int64_t n, float lr, float wd, cudaStream_t st) {
  if (n < 0) return set_error(ASTRA_ERR_CONFIG, "dense_sgd: bad size");
  if (n == 0) return ASTRA_OK;
  dense_sgd_kernel<<<grid_for(n), kDenseThreads, 0, st>>>(W, grads, n, lr, wd);
  ASTRA_LAUNCHED("dense_sgd");
  return ASTRA_OK;
}

}  // namespace astra
