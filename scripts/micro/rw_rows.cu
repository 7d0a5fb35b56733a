// Microbenchmark: the DRAM ceiling for the step's access pattern -- read and
// write back U random, distinct 3 KB rows (d = 768 fp32) of a 4 GB matrix.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int UNR>
__global__ void __launch_bounds__(256) rw_kernel(float* W, const int* rows, int U) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int u0 = warp * UNR; u0 < U; u0 += nw * UNR) {
    float4 v[UNR][6];
#pragma unroll
    for (int k = 0; k < UNR; ++k) {
      if (u0 + k < U) {
        const float4* p = reinterpret_cast<const float4*>(W + (size_t)rows[u0 + k] * 768) + lane;
#pragma unroll
        for (int q = 0; q < 6; ++q) v[k][q] = p[q * 32];
      }
    }
#pragma unroll
    for (int k = 0; k < UNR; ++k) {
      if (u0 + k < U) {
        float4* p = reinterpret_cast<float4*>(W + (size_t)rows[u0 + k] * 768) + lane;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          float4 x = v[k][q];
          x.x += 1.f; x.y += 1.f; x.z += 1.f; x.w += 1.f;
          p[q * 32] = x;
        }
      }
    }
  }
}

int main() {
  const int L = 1305265, U = 480000;
  float* W; int* rows;
  cudaMalloc(&W, sizeof(float) * (size_t)L * 768);
  cudaMemset(W, 0, sizeof(float) * (size_t)L * 768);
  std::vector<int> h(L);
  for (int i = 0; i < L; ++i) h[i] = i;
  std::mt19937 g(1);
  std::shuffle(h.begin(), h.end(), g);
  h.resize(U);
  std::sort(h.begin(), h.end());  // ascending like the sorted unique-label list
  cudaMalloc(&rows, sizeof(int) * U);
  cudaMemcpy(rows, h.data(), sizeof(int) * U, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {148 * 4, 148 * 8}) {
    for (int unr : {1, 2, 4}) {
      auto run = [&]() {
        if (unr == 1) rw_kernel<1><<<grid, 256>>>(W, rows, U);
        else if (unr == 2) rw_kernel<2><<<grid, 256>>>(W, rows, U);
        else rw_kernel<4><<<grid, 256>>>(W, rows, U);
      };
      for (int i = 0; i < 3; ++i) run();
      cudaEventRecord(a);
      for (int i = 0; i < 10; ++i) run();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      printf("grid %d unr %d: %.3f ms  %.0f GB/s (read+write)\n", grid, unr, ms, 2.0 * U * 3072 / ms / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
