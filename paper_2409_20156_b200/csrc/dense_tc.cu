// dense_tc.cu — fp32-accurate GEMM D = A B^T on the tf32 tensor cores
// (3xTF32), for the all-negatives arm (trainer.py:593-606: scores = E W^T,
// grad_emb = G W, grad_W = G^T E) in place of fp32 SIMT SGEMM.
//
// Each fp32 operand x is split into x_hi = x with the low 13 mantissa bits
// cleared (exactly representable in tf32) and x_lo = x - x_hi (exact in fp32),
// and D = A_hi B_hi^T + A_lo B_hi^T + A_hi B_lo^T accumulates in fp32 in TMEM:
// the dropped A_lo B_lo^T term and the tf32 truncation of the lo parts are
// ~2^-22 of each product, below fp32's own rounding of the sum.
//
//   split_kernel   A [M, K] (or given as [K, M]) -> A_hi, A_lo [M, Kp] K-major
//                  (Kp = K rounded up to 32, zero padded); 32 x 32 tiles
//                  through shared memory, so transposed inputs stay coalesced.
//   gemm_kernel    CTA pairs (tcgen05.mma.cta_group::2.kind::tf32, M = 256
//                  rows x N = 256 columns per MMA, fp32 accumulators in TMEM,
//                  2 x 256 columns double-buffered against the epilogue),
//                  operands TMA-loaded (SWIZZLE_128B, 32 tf32 per 128-byte
//                  row = 4 MMAs of K = 8 per stage) into a 6-stage ring: the
//                  refresh kernel's pipeline (refresh_tc.cu) with a store
//                  epilogue. The K sweep runs the three (A, B) pairs one
//                  after the other; units = (row-tile pair, column tile,
//                  K part) over a persistent grid; with K parts > 1 each part
//                  writes a partial tile and reduce_kernel sums the parts in
//                  order (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace astra {
namespace {

constexpr int BM = 128, BN = 256, BKE = 32, NST = 6;  // BKE: tf32 elements per 128-byte row
constexpr int A_ST = BM * 128, B_ST = (BN / 2) * 128, STG = A_ST + B_ST;
constexpr int kEpiWarp0 = 4, kEpiWarps = 4, kThreads = 32 * (kEpiWarp0 + kEpiWarps);
constexpr int TMEM_COLS = 512;
constexpr size_t kSmem = 1024 + NST * STG + 256;
// idesc kind::tf32: D = F32 (bits 4-5 = 1), A = B = TF32 (format 2 at [7,10) and
// [10,13)), both K-major, N >> 3 at [17,23), M >> 4 at [24,29); M = 256 (pair)
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(256 >> 4) << 24);

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ uint64_t sdesc(const void* p) {  // K-major SWIZZLE_128B, SBO 1024 B, sm_100 version 1
  const uint32_t a = smem_u32(p);
  return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}
__device__ __forceinline__ void tma_pair(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct GemmArgs {
  int64_t M, N;
  int nkb;            // 32-element K blocks per operand pair (Kp / 32)
  int n_mt, n_nt;     // row-tile pairs (256 rows), column tiles (256)
  int kparts, kb_per_part;  // K parts over the 3 * nkb blocks of the sweep
  float* out;         // [kparts][M][N] (kparts == 1: D itself)
};

// K block j of the sweep (0 <= j < 3 nkb): pair s = j / nkb of
// (A_hi, B_hi), (A_lo, B_hi), (A_hi, B_lo), column block j % nkb.
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tAh, const __grid_constant__ CUtensorMap tAl,
                const __grid_constant__ CUtensorMap tBh, const __grid_constant__ CUtensorMap tBl, GemmArgs g) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = ctarank();
  const bool leader = crank == 0;
  const int64_t cluster = blockIdx.x / 2, n_clusters = gridDim.x / 2;
  extern __shared__ __align__(1024) unsigned char dsm_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;
  unsigned char* sB = smem + NST * A_ST;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STG);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  const int64_t n_units = static_cast<int64_t>(g.n_mt) * g.n_nt * g.kparts;
  const int total_kb = 3 * g.nkb;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;
  // unit u: K part kp = u / (n_mt n_nt), column tile nt, row-tile pair mt (mt fastest:
  // concurrent clusters share the column tile's B rows in L2)
  auto unit = [&](int64_t u, int& mt, int& nt, int& kb0, int& kb1) {
    const int64_t t = u % (static_cast<int64_t>(g.n_mt) * g.n_nt);
    const int kp = static_cast<int>(u / (static_cast<int64_t>(g.n_mt) * g.n_nt));
    mt = static_cast<int>(t % g.n_mt);
    nt = static_cast<int>(t / g.n_mt);
    kb0 = std::min(total_kb, kp * g.kb_per_part);
    kb1 = std::min(total_kb, kb0 + g.kb_per_part);
  };
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs: own A rows, own half of the B tile)
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = cluster; u < n_units; u += n_clusters) {
        int mt, nt, kb0, kb1;
        unit(u, mt, nt, kb0, kb1);
        const int r0 = mt * 2 * BM + static_cast<int>(crank) * BM;
        const int c0 = nt * BN + static_cast<int>(crank) * (BN / 2);
        for (int j = kb0; j < kb1; ++j) {
          const int s = j / g.nkb, kc = (j - s * g.nkb) * BKE;
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t bar = mapa(&full[stage], 0);
          if (leader) mbar_expect_tx(&full[stage], 2 * STG);
          tma_pair(sA + stage * A_ST, s == 1 ? &tAl : &tAh, bar, kc, r0);
          tma_pair(sB + stage * B_ST, s == 2 ? &tBl : &tBh, bar, kc, c0);
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && leader) {  // ---- MMA issuer (the pair's even CTA)
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int64_t u = cluster; u < n_units; u += n_clusters) {
      int mt, nt, kb0, kb1;
      unit(u, mt, nt, kb0, kb1);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dcol = tmem_base + static_cast<uint32_t>(acc * BN);
      for (int j = kb0; j < kb1; ++j) {
        mbar_wait(&full[stage], phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint64_t ad = sdesc(sA + stage * A_ST), bd = sdesc(sB + stage * B_ST);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_tf32(dcol, ad + 2 * kk, bd + 2 * kk, (j > kb0 || kk) ? 1u : 0u);
          commit_pair(&empty[stage]);
        }
        __syncwarp();
        if (++stage == NST) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) commit_pair(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= kEpiWarp0) {  // ---- epilogue: TMEM -> fp32 tile rows
    const int e = warp - kEpiWarp0;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(e * 32) << 16);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t u = cluster; u < n_units; u += n_clusters) {
      int mt, nt, kb0, kb1;
      unit(u, mt, nt, kb0, kb1);
      const int kp = static_cast<int>(u / (static_cast<int64_t>(g.n_mt) * g.n_nt));
      mbar_wait(&tfull[acc], acc_phase);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t row = static_cast<int64_t>(mt) * 2 * BM + crank * BM + e * 32 + lane;
      float* orow = g.out + (static_cast<int64_t>(kp) * g.M + row) * g.N;
      const bool vec = (g.N & 3) == 0;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        __syncwarp();
        tmem_ld32(lane_base + static_cast<uint32_t>(acc * BN + c), r);
        const int64_t col = static_cast<int64_t>(nt) * BN + c;
        if (row < g.M && col < g.N) {
          if (vec && col + 32 <= g.N) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(orow + col + i) =
                  make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]), __uint_as_float(r[i + 2]),
                              __uint_as_float(r[i + 3]));
          } else {
            for (int i = 0; i < 32 && col + i < g.N; ++i) orow[col + i] = __uint_as_float(r[i]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(&tempty[acc], 0))
                     : "memory");
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// hi / lo split of a [R, K] operand into K-major [R, Kp] arrays (zero padded).
// kmajor: the source is [R, K] row-major; else it is [K, R] row-major.
// 32 x 32 tiles, 32 x 8 threads.
__global__ void __launch_bounds__(256) split_kernel(const float* __restrict__ src, int kmajor, int64_t R, int64_t K,
                                                    int64_t Kp, float* __restrict__ hi, float* __restrict__ lo) {
  __shared__ float t[32][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32, k0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8) {
    float v = 0.0f;
    if (kmajor) {  // t[row][k]: coalesced along k
      const int64_t r = r0 + i, k = k0 + tx;
      if (r < R && k < K) v = src[r * K + k];
      t[i][tx] = v;
    } else {  // source [K, R]: coalesced along r, transposed through the tile
      const int64_t k = k0 + i, r = r0 + tx;
      if (r < R && k < K) v = src[k * R + r];
      t[tx][i] = v;
    }
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, k = k0 + tx;
    if (r < R && k < Kp) {
      const float x = t[i][tx];
      const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
      hi[r * Kp + k] = h;
      lo[r * Kp + k] = __fsub_rn(x, h);
    }
  }
}

// The K-major case with K % 4 == 0: a straight vectorised map (16-byte loads
// and stores, no shared-memory tile), zero padding past K.
__global__ void __launch_bounds__(256) split_kmajor_v4_kernel(const float4* __restrict__ src, int64_t R, int64_t K4,
                                                              int64_t Kp4, float4* __restrict__ hi,
                                                              float4* __restrict__ lo) {
  const int64_t n = R * Kp4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / Kp4, k4 = i - r * Kp4;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k4 < K4) x = src[r * K4 + k4];
    float4 h;
    h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
    h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
    h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
    h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
    hi[i] = h;
    lo[i] = make_float4(__fsub_rn(x.x, h.x), __fsub_rn(x.y, h.y), __fsub_rn(x.z, h.z), __fsub_rn(x.w, h.w));
  }
}

// D[i] = sum over parts p of part[p][i], in part order.
__global__ void __launch_bounds__(256) reduce_kernel(const float* __restrict__ part, int kparts, int64_t n,
                                                     float* __restrict__ D) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = part[i];
    for (int p = 1; p < kparts; ++p) s = __fadd_rn(s, part[static_cast<int64_t>(p) * n + i]);
    D[i] = s;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_map_f32(CUtensorMap* m, const float* base, int64_t rows, int64_t Kp, int box_rows) {
  auto fn = encode();
  if (!fn) return set_error(ASTRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kp) * 4};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BKE), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ASTRA_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (%d)", static_cast<int>(r));
  return ASTRA_OK;
}

// K parts: the fewest that keep >= 93% of the SM pairs busy over whole rounds
// (at most 64, at least 8 K blocks each).
int gemm_kparts(int64_t tiles, int total_kb, int n_cl) {
  int best = 1;
  double best_eff = -1.0;
  for (int p = 1; p <= 64 && p <= std::max(1, total_kb / 8); ++p) {
    const int64_t units = tiles * p;
    const int64_t rounds = (units + n_cl - 1) / n_cl;
    const double eff = static_cast<double>(units) / static_cast<double>(rounds * n_cl);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = p;
    }
    if (best_eff >= 0.93) break;
  }
  return best;
}

struct GemmPlan {
  int64_t Kp;
  int nkb, n_mt, n_nt, kparts, kb_per_part, grid;
};

GemmPlan plan_gemm(int64_t M, int64_t N, int64_t K) {
  GemmPlan p;
  p.Kp = (K + BKE - 1) / BKE * BKE;
  p.nkb = static_cast<int>(p.Kp / BKE);
  p.n_mt = static_cast<int>((M + 2 * BM - 1) / (2 * BM));
  p.n_nt = static_cast<int>((N + BN - 1) / BN);
  const int n_cl = std::max(1, num_sms() / 2);
  const int64_t tiles = static_cast<int64_t>(p.n_mt) * p.n_nt;
  p.kparts = gemm_kparts(tiles, 3 * p.nkb, n_cl);
  // no empty parts: kb_per_part = ceil(3 nkb / kparts), then as many parts as that needs
  p.kb_per_part = (3 * p.nkb + p.kparts - 1) / p.kparts;
  p.kparts = (3 * p.nkb + p.kb_per_part - 1) / p.kb_per_part;
  p.grid = static_cast<int>(std::min<int64_t>(n_cl, tiles * p.kparts)) * 2;
  return p;
}

}  // namespace

size_t gemm_f32_workspace(int64_t M, int64_t N, int64_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 256;
  const GemmPlan p = plan_gemm(M, N, K);
  Carve c(nullptr, 0);
  c.take<float>(static_cast<size_t>(M) * p.Kp);  // A hi, lo
  c.take<float>(static_cast<size_t>(M) * p.Kp);
  c.take<float>(static_cast<size_t>(N) * p.Kp);  // B hi, lo
  c.take<float>(static_cast<size_t>(N) * p.Kp);
  if (p.kparts > 1) c.take<float>(static_cast<size_t>(p.kparts) * M * N);
  return c.off + 256;
}

int gemm_f32(const float* A, int a_kmajor, const float* B, int b_kmajor, int64_t M, int64_t N, int64_t K, float* D,
             void* ws, size_t ws_bytes, cudaStream_t st) {
  if (M < 0 || N < 0 || K < 0) return set_error(ASTRA_ERR_CONFIG, "gemm_f32: negative shape");
  if (M == 0 || N == 0) return ASTRA_OK;
  if (K == 0) return check_cuda(cudaMemsetAsync(D, 0, sizeof(float) * M * N, st), "gemm_f32 memset");
  if (M > (int64_t(1) << 31) || N > (int64_t(1) << 31)) return set_error(ASTRA_ERR_CONFIG, "gemm_f32: shape too large");
  const GemmPlan p = plan_gemm(M, N, K);
  if (!ws || ws_bytes < gemm_f32_workspace(M, N, K))
    return set_error(ASTRA_ERR_CONFIG, "gemm_f32 workspace too small (%zu < %zu)", ws_bytes, gemm_f32_workspace(M, N, K));
  Carve c(ws, ws_bytes);
  float* Ah = c.take<float>(static_cast<size_t>(M) * p.Kp);
  float* Al = c.take<float>(static_cast<size_t>(M) * p.Kp);
  float* Bh = c.take<float>(static_cast<size_t>(N) * p.Kp);
  float* Bl = c.take<float>(static_cast<size_t>(N) * p.Kp);
  float* part = p.kparts > 1 ? c.take<float>(static_cast<size_t>(p.kparts) * M * N) : D;
  if (p.Kp / 32 > 65535) return set_error(ASTRA_ERR_CONFIG, "gemm_f32: K too large (%lld)", static_cast<long long>(K));
  auto split = [&](const float* X, int kmajor, int64_t R, float* hi, float* lo) {
    if (kmajor && K % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) {
      const int64_t n = R * (p.Kp / 4);
      split_kmajor_v4_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 16LL * num_sms())), 256, 0,
                               st>>>(reinterpret_cast<const float4*>(X), R, K / 4, p.Kp / 4,
                                     reinterpret_cast<float4*>(hi), reinterpret_cast<float4*>(lo));
    } else {
      split_kernel<<<dim3(static_cast<unsigned>((R + 31) / 32), static_cast<unsigned>(p.Kp / 32)), 256, 0, st>>>(
          X, kmajor, R, K, p.Kp, hi, lo);
    }
  };
  split(A, a_kmajor, M, Ah, Al);
  ASTRA_LAUNCHED("gemm_split");
  split(B, b_kmajor, N, Bh, Bl);
  ASTRA_LAUNCHED("gemm_split");
  CUtensorMap tAh, tAl, tBh, tBl;
  ASTRA_TRY(make_map_f32(&tAh, Ah, M, p.Kp, BM));
  ASTRA_TRY(make_map_f32(&tAl, Al, M, p.Kp, BM));
  ASTRA_TRY(make_map_f32(&tBh, Bh, N, p.Kp, BN / 2));
  ASTRA_TRY(make_map_f32(&tBl, Bl, N, p.Kp, BN / 2));
  GemmArgs g;
  g.M = M;
  g.N = N;
  g.nkb = p.nkb;
  g.n_mt = p.n_mt;
  g.n_nt = p.n_nt;
  g.kparts = p.kparts;
  g.kb_per_part = p.kb_per_part;
  g.out = part;
  static bool attr = false;
  if (!attr) {
    ASTRA_TRY(check_cuda(cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem)),
                         "gemm smem attr"));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(p.grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  {
    KernelTimer kt("gemm_f32", st);
    ASTRA_TRY(check_cuda(cudaLaunchKernelEx(&cfg, gemm_kernel, tAh, tAl, tBh, tBl, g), "launch gemm_f32"));
    ASTRA_LAUNCHED("gemm_f32");
  }
  if (p.kparts > 1) {
    const int64_t n = M * N;
    reduce_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 8LL * num_sms())), 256, 0, st>>>(
        part, p.kparts, n, D);
    ASTRA_LAUNCHED("gemm_reduce");
  }
  return ASTRA_OK;
}

}  // namespace astra
