// capi.cu — the extern "C" boundary (include/astra_b200.h) and host helpers.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "refresh_tc.cuh"
#include "topk.cuh"

namespace astra {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ASTRA_OK;
  return set_error(ASTRA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static std::atomic<bool> g_kt_on{false};
static std::mutex g_kt_mu;
static std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> g_kt;

bool kernel_timing_on() { return g_kt_on.load(std::memory_order_relaxed); }

// Timing events come from a pool filled when timing is enabled, so no
// cudaEventCreate runs between the launches being timed (event creation can
// block the host for milliseconds when the driver grows its event storage).
static std::vector<cudaEvent_t> g_kt_pool;
static constexpr size_t kKtPool = 8192;

cudaEvent_t kernel_timing_event() {
  {
    std::lock_guard<std::mutex> lk(g_kt_mu);
    if (!g_kt_pool.empty()) {
      cudaEvent_t e = g_kt_pool.back();
      g_kt_pool.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void kernel_timing_push(const char* name, cudaEvent_t e0, cudaEvent_t e1) {
  std::lock_guard<std::mutex> lk(g_kt_mu);
  g_kt[name].emplace_back(e0, e1);
}

int num_sms() {
  static thread_local int dev_cached = -1, sms_cached = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != dev_cached) {
    cudaDeviceGetAttribute(&sms_cached, cudaDevAttrMultiProcessorCount, dev);
    dev_cached = dev;
    if (sms_cached <= 0) sms_cached = 148;
  }
  return sms_cached;
}

// defined in the kernel translation units
int f32_to_bf16(const float*, uint16_t*, int64_t, cudaStream_t);
size_t refresh_workspace_size(int64_t, int64_t, int, int, int);
int refresh_topk(const float*, const uint16_t*, int64_t, int, const float*, const uint16_t*, const uint8_t*, int64_t,
                 int64_t, const int64_t*, const int32_t*, int, int, uint64_t*, int32_t*, float*, void*, size_t,
                 cudaStream_t);
int quantize_e4m3(const void*, int, int64_t, uint8_t*, float*, cudaStream_t);
int topk_merge(const uint64_t*, int64_t, int, int, int, uint64_t*, int32_t*, float*, uint64_t*, cudaStream_t);
int refresh_flagged(const void*, size_t, int64_t, int64_t, int, int, int, int64_t*, cudaStream_t);
int sample_slates(uint64_t, uint32_t, uint32_t, const int64_t*, int, const int64_t*, const int32_t*, const int32_t*,
                  int, int, const int32_t*, const float*, int, int, int, int64_t, int, int, int32_t*, int8_t*,
                  int8_t*, float*, cudaStream_t);
int importance_split(const int32_t*, const float*, int64_t, int, int, int32_t*, int32_t*, float*, cudaStream_t);
size_t step_workspace_size(int, int, int, int64_t);
void set_step_deterministic(int on);
size_t dense_workspace_size(int B);
int dense_bce(const void* S, int s_f64, int B, int64_t L, const int64_t* pos_indptr, const int32_t* pos_ids,
              float* G, double* loss_out, void* workspace, size_t ws_bytes, cudaStream_t st);
int dense_sgd(float* W, const float* grads, int64_t n, float lr, float wd, cudaStream_t st);
size_t gemm_f32_workspace(int64_t M, int64_t N, int64_t K);
int refresh_plan_j(int64_t nq, int64_t L, int d, int k);
int refresh_sharded_stage(int stage, const float* qf, const uint16_t* qb, int64_t nq, int d, const uint16_t* wb,
                          int64_t L, int64_t off, const int64_t* pos_indptr, const int32_t* pos_ids, int k,
                          uint32_t* sample_top, const uint64_t* tau_keys, uint64_t* io_keys, int32_t* counts,
                          int32_t* flags, void* ws, size_t ws_bytes, cudaStream_t st);
int rerank_only(const float* qf, int64_t nq, int d, const uint64_t* cand, int kc, const void* labels, int w_dtype,
                int64_t off, int k, uint64_t* out_keys, int32_t* out_ids, float* out_scores, cudaStream_t st);
int gemm_f32(const float* A, int a_kmajor, const float* B, int b_kmajor, int64_t M, int64_t N, int64_t K, float* D,
             void* ws, size_t ws_bytes, cudaStream_t st);
int slate_step(const float*, const float*, const int32_t*, const int8_t*, const int8_t*, int64_t, const float*,
               int64_t, const float*, int, int, int, void*, int, float*, float*, int, int64_t, int64_t, double, double,
               double, double, double, int64_t, float*, double*, int32_t*, float*, float*, void*, size_t, cudaStream_t);
int apply_updates(void*, int, int64_t, int, const int64_t*, const float*, int64_t, float, float, int32_t*,
                  cudaStream_t);

}  // namespace astra

using namespace astra;

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

const char* astra_version(void) { return "astra-b200 0.1 (sm_100a)"; }
const char* astra_last_error(void) { return g_err; }
uint64_t astra_launch_count(void) { return g_launches.load(); }

void astra_kernel_timing_enable(int on) {
  if (on) {
    std::lock_guard<std::mutex> lk(g_kt_mu);
    while (g_kt_pool.size() < kKtPool) {
      cudaEvent_t e = nullptr;
      if (cudaEventCreate(&e) != cudaSuccess) break;
      g_kt_pool.push_back(e);
    }
  }
  g_kt_on.store(on != 0);
}

void astra_set_refresh_sm_budget(int n_sms) { set_refresh_sm_budget(n_sms); }
void astra_set_step_deterministic(int on) { set_step_deterministic(on); }

int astra_kernel_timing(const char* name, double* total_ms, int64_t* count) {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  {
    std::lock_guard<std::mutex> lk(g_kt_mu);
    auto it = g_kt.find(name);
    if (it != g_kt.end()) ev.swap(it->second);
  }
  double tot = 0.0;
  for (auto& p : ev) {
    ASTRA_TRY(check_cuda(cudaEventSynchronize(p.second), "kernel timing sync"));
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, p.first, p.second);
    tot += ms;
  }
  {
    std::lock_guard<std::mutex> lk(g_kt_mu);  // back to the pool
    for (auto& p : ev) {
      g_kt_pool.push_back(p.first);
      g_kt_pool.push_back(p.second);
    }
  }
  if (total_ms) *total_ms = tot;
  if (count) *count = static_cast<int64_t>(ev.size());
  return ASTRA_OK;
}

int astra_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  ASTRA_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  if (sm_count) ASTRA_TRY(check_cuda(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev), "attr"));
  if (cc_major) ASTRA_TRY(check_cuda(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev), "attr"));
  if (cc_minor) ASTRA_TRY(check_cuda(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev), "attr"));
  return ASTRA_OK;
}

int astra_f32_to_bf16(const float* src, uint16_t* dst, int64_t n, void* stream) {
  return f32_to_bf16(src, dst, n, S(stream));
}

size_t astra_refresh_workspace_size(int64_t nq, int64_t n_labels, int d, int k, int mode) {
  return refresh_workspace_size(nq, n_labels, d, k, mode);
}

int astra_refresh_topk(const float* queries_f32, const uint16_t* queries_bf16, int64_t nq, int d,
                       const float* labels_f32, const uint16_t* labels_bf16, const uint8_t* labels_e4m3,
                       int64_t n_labels, int64_t label_offset, const int64_t* pos_indptr, const int32_t* pos_ids,
                       int k, int mode, uint64_t* out_keys, int32_t* out_ids, float* out_scores, void* workspace,
                       size_t workspace_bytes, void* stream) {
  return refresh_topk(queries_f32, queries_bf16, nq, d, labels_f32, labels_bf16, labels_e4m3, n_labels, label_offset,
                      pos_indptr, pos_ids, k, mode, out_keys, out_ids, out_scores, workspace, workspace_bytes,
                      S(stream));
}

int astra_quantize_e4m3(const void* src, int src_bf16, int64_t n, uint8_t* dst, float* scratch, void* stream) {
  return quantize_e4m3(src, src_bf16, n, dst, scratch, S(stream));
}

int astra_refresh_flagged(const void* workspace, size_t workspace_bytes, int64_t nq, int64_t n_labels, int d, int k,
                          int mode, int64_t* out_count, void* stream) {
  return refresh_flagged(workspace, workspace_bytes, nq, n_labels, d, k, mode, out_count, S(stream));
}

size_t astra_merge_workspace_size(int64_t nq, int k_out) {
  return static_cast<size_t>(nq) * (topk_cap(k_out) + kTopkSlack) * sizeof(uint64_t);
}

int astra_topk_merge(const uint64_t* part_keys, int64_t nq, int n_parts, int k_in, int k_out, uint64_t* out_keys,
                     int32_t* out_ids, float* out_scores, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_parts < 1 || k_in < 1 || k_out < 1 || k_out > 2048) return set_error(ASTRA_ERR_CONFIG, "merge: bad sizes");
  if (!workspace || workspace_bytes < astra_merge_workspace_size(nq, k_out))
    return set_error(ASTRA_ERR_CONFIG, "merge workspace too small");
  return topk_merge(part_keys, nq, n_parts, k_in, k_out, out_keys, out_ids, out_scores,
                    static_cast<uint64_t*>(workspace), S(stream));
}

int astra_importance_split(const int32_t* ids, const float* scores, int64_t nq, int k_tot, int k_h, int32_t* hard,
                           int32_t* cand, float* cand_q, void* stream) {
  return importance_split(ids, scores, nq, k_tot, k_h, hard, cand, cand_q, S(stream));
}

int astra_sample_slates(uint64_t seed, uint32_t epoch, uint32_t step, const int64_t* rows, int B,
                        const int64_t* pos_indptr, const int32_t* pos_ids, const int32_t* hard, int hard_stride,
                        int k_h, const int32_t* cand, const float* cand_q, int cand_stride, int n_c, int k_i,
                        int64_t n_labels, int k_p, int k_r, int32_t* ids, int8_t* y, int8_t* origin, float* weights,
                        void* stream) {
  return sample_slates(seed, epoch, step, rows, B, pos_indptr, pos_ids, hard, hard_stride, k_h, cand, cand_q,
                       cand_stride, n_c, k_i, n_labels, k_p, k_r, ids, y, origin, weights, S(stream));
}

size_t astra_step_workspace_size(int B, int S_, int d, int64_t n_labels_local) {
  return step_workspace_size(B, S_, d, n_labels_local);
}

int astra_slate_step(const float* emb, const float* keep, const int32_t* ids, const int8_t* y, const int8_t* origin,
                     int64_t origin_row_stride, const float* weights, int64_t weights_row_stride,
                     const float* factors_in, int B, int S_, int d, void* W, int w_dtype, float* adam_m,
                     float* adam_v, int optimizer, int64_t n_labels_local, int64_t label_offset, double lr,
                     double weight_decay, double adam_beta1, double adam_beta2, double adam_eps, int64_t adam_step,
                     float* grad_emb, double* loss_out, int32_t* status, float* factors_out, float* w_absmax,
                     void* workspace, size_t workspace_bytes, void* stream) {
  return slate_step(emb, keep, ids, y, origin, origin_row_stride, weights, weights_row_stride, factors_in, B, S_, d,
                    W, w_dtype, adam_m, adam_v, optimizer, n_labels_local, label_offset, lr, weight_decay,
                    adam_beta1, adam_beta2, adam_eps, adam_step, grad_emb, loss_out, status, factors_out, w_absmax,
                    workspace, workspace_bytes, S(stream));
}

int astra_apply_updates(void* W, int w_dtype, int64_t n_labels, int d, const int64_t* ids, const float* grads,
                        int64_t U, float lr, float weight_decay, int32_t* status, void* stream) {
  return apply_updates(W, w_dtype, n_labels, d, ids, grads, U, lr, weight_decay, status, S(stream));
}

size_t astra_dense_workspace_size(int B) { return dense_workspace_size(B); }

int astra_dense_bce(const void* scores, int scores_f64, int B, int64_t n_labels, const int64_t* pos_indptr,
                    const int32_t* pos_ids, float* G, double* loss_out, void* workspace, size_t workspace_bytes,
                    void* stream) {
  return dense_bce(scores, scores_f64, B, n_labels, pos_indptr, pos_ids, G, loss_out, workspace, workspace_bytes,
                   S(stream));
}

int astra_dense_sgd(float* W, const float* grads, int64_t n, float lr, float weight_decay, void* stream) {
  return dense_sgd(W, grads, n, lr, weight_decay, S(stream));
}

int astra_refresh_plan_j(int64_t nq, int64_t n_labels, int d, int k) { return refresh_plan_j(nq, n_labels, d, k); }

int astra_refresh_sharded_stage(int stage, const float* queries_f32, const uint16_t* queries_bf16, int64_t nq, int d,
                                const uint16_t* labels_bf16, int64_t n_labels, int64_t label_offset,
                                const int64_t* pos_indptr, const int32_t* pos_ids, int k, uint32_t* sample_top,
                                const uint64_t* tau_keys, uint64_t* io_keys, int32_t* counts, int32_t* flags,
                                void* workspace, size_t workspace_bytes, void* stream) {
  return refresh_sharded_stage(stage, queries_f32, queries_bf16, nq, d, labels_bf16, n_labels, label_offset,
                               pos_indptr, pos_ids, k, sample_top, tau_keys, io_keys, counts, flags, workspace,
                               workspace_bytes, S(stream));
}

int astra_rerank_candidates(const float* queries, int64_t nq, int d, const uint64_t* cand, int kc, const void* labels,
                            int w_dtype, int64_t label_offset, int k, uint64_t* out_keys, int32_t* out_ids,
                            float* out_scores, void* stream) {
  return rerank_only(queries, nq, d, cand, kc, labels, w_dtype, label_offset, k, out_keys, out_ids, out_scores,
                     S(stream));
}

size_t astra_gemm_f32_workspace_size(int64_t M, int64_t N, int64_t K) { return gemm_f32_workspace(M, N, K); }

int astra_gemm_f32(const float* A, int a_kmajor, const float* B, int b_kmajor, int64_t M, int64_t N, int64_t K,
                   float* D, void* workspace, size_t workspace_bytes, void* stream) {
  return gemm_f32(A, a_kmajor, B, b_kmajor, M, N, K, D, workspace, workspace_bytes, S(stream));
}

int astra_stream_sync(void* stream) { return check_cuda(cudaStreamSynchronize(S(stream)), "stream sync"); }

}  // extern "C"
