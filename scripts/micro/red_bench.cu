// Microbenchmark: throughput of vector fp32 reductions (red.global.add.v4.f32)
// into a B x d (1024 x 768) L2-resident buffer from n_slots random rows, as the
// label-major single-pass step would issue for grad_emb.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void red_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

__global__ void red_kernel(float* ge, const int* rows, int n, int d) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < n; s += nw) {
    float* p = ge + (size_t)rows[s] * d;
    for (int c = lane * 4; c < d; c += 128) red_v4(p + c, make_float4(1.f, 1.f, 1.f, 1.f));
  }
}

__global__ void red_scalar_kernel(float* ge, const int* rows, int n, int d) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < n; s += nw) {
    float* p = ge + (size_t)rows[s] * d;
    for (int c = lane; c < d; c += 32) atomicAdd(p + c, 1.f);
  }
}

__global__ void red_u64_kernel(unsigned long long* ge, const int* rows, int n, int d) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < n; s += nw) {
    unsigned long long* p = ge + (size_t)rows[s] * d;
    for (int c = lane; c < d; c += 32) {
      double v = (double)(s & 7) * 1.25 * 4503599627370496.0;
      asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p + c), "l"((long long)__double2ll_rn(v)) : "memory");
    }
  }
}

int main() {
  const int B = 1024, d = 768, n = 1024 * 584;
  float* ge; int* rows;
  cudaMalloc(&ge, sizeof(float) * B * d);
  cudaMalloc(&rows, sizeof(int) * n);
  int* h = new int[n];
  uint32_t x = 12345;
  for (int i = 0; i < n; ++i) { x = x * 1664525u + 1013904223u; h[i] = (x >> 8) % B; }
  cudaMemcpy(rows, h, sizeof(int) * n, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  unsigned long long* ge64;
  cudaMalloc(&ge64, 8ull * B * d);
  for (int variant = 0; variant < 3; ++variant)
  for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
    for (int it = 0; it < 3; ++it) {
      if (variant == 0) red_kernel<<<grid, 256>>>(ge, rows, n, d); else if (variant == 1) red_scalar_kernel<<<grid, 256>>>(ge, rows, n, d); else red_u64_kernel<<<grid, 256>>>(ge64, rows, n, d);
    }
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) {
      if (variant == 0) red_kernel<<<grid, 256>>>(ge, rows, n, d); else if (variant == 1) red_scalar_kernel<<<grid, 256>>>(ge, rows, n, d); else red_u64_kernel<<<grid, 256>>>(ge64, rows, n, d);
    }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%s grid %d: %.3f ms  %.1f G fp32-adds/s\n", variant == 2 ? "u64" : variant ? "scalar" : "v4", grid, ms, (double)n * d / ms / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
