// refresh_tc.cu — bf16 tcgen05 GEMM of queries x labels with a fused top-k
// epilogue: the B200 shortlist refresh (replaces anns.py:253-256).
//
// One CTA owns a 128-query tile and sweeps a contiguous range of label tiles
// (N = 256 labels each). Warp roles (256 threads):
//   warp 0      TMA producer: A (128 x 64 bf16) and B (256 x 64 bf16) k-blocks,
//               SWIZZLE_128B, into a 4-stage shared-memory ring (48 KB/stage).
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.kind::f16
//               (M=128, N=256, K=16) into a TMEM accumulator; tcgen05.commit
//               releases smem stages and publishes finished accumulators.
//   warp 2      TMEM allocator (512 columns = 2 accumulators of 256 fp32 cols).
//   warps 4-7   epilogue: tcgen05.ld 32 columns at a time (thread = query row =
//               TMEM lane), running top-k per query (topk.cuh). The two TMEM
//               accumulators double-buffer the epilogue against the next MMA.
// Scores never leave the SM; per-query partial top-k lists go to HBM once.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "topk.cuh"

namespace astra {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, UMMA_K = 16, STAGES = 4;
constexpr int A_STAGE = BM * BK * 2;  // 16 KB
constexpr int B_STAGE = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
constexpr int TMEM_COLS = 512;
constexpr int kEpiWarp0 = 4;
// SPLIT = epilogue warps per TMEM lane quadrant; each owns (32 query rows) x
// (BN / SPLIT columns) and its own partial list. Threads = 32 * (4 + 4*SPLIT).
template <int SPLIT>
constexpr int threads_for() { return 32 * (kEpiWarp0 + 4 * SPLIT); }
constexpr size_t kSmemBytes = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256 /*barriers*/;

// idesc for kind::f16: D=F32, A=B=BF16, both K-major, N>>3 at [17,23), M>>4 at [24,29)
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)  // suspend-time hint: sleep until the phase flips
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Multicast variant: the box lands at the same smem offset in every CTA of
// `mask` and completes tx bytes on the mbarrier at the same offset in each.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (8-row x 128 B atoms,
// SBO = 1024 B between atoms, version 1 for sm_100).
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint32_t a = smem_u32(p);
  return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Arrive on `bar` (same smem offset) in every CTA of `mask` once this thread's
// prior tcgen05.mma ops complete: releases a multicast-filled stage cluster-wide.
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// Issue one 32-column TMEM load without waiting (pair with tmem_wait()).
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// r[j] for a run-time j without local memory: a 5-level select tree.
__device__ __forceinline__ uint32_t pick32(const uint32_t* r, int j) {
  uint32_t a[16], b[8], c[4], d[2];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = (j & 16) ? r[i + 16] : r[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = (j & 8) ? a[i + 8] : a[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = (j & 4) ? b[i + 4] : b[i];
#pragma unroll
  for (int i = 0; i < 2; ++i) d[i] = (j & 2) ? c[i + 2] : c[i];
  return (j & 1) ? d[1] : d[0];
}

struct TcArgs {
  int64_t nq, L, off;
  int d, k, cap;
  int64_t n_lt, tiles_per_part;  // label tiles; label tiles per part
  const int64_t* pos_indptr;
  const int32_t* pos_ids;
  uint64_t* bufs;
  uint64_t* part_keys;
  uint64_t* gtau;  // nq shared thresholds (zeroed by the host before launch)
  int debug_no_topk;  // ASTRA_TC_DEBUG_NO_TOPK=1: skip selection (pipeline-rate measurement only)
  unsigned long long* dbg;  // ASTRA_TC_DEBUG_COUNTERS=1: [slow chunks, candidates, compactions, chunks]
};

// Schedule: grid (query tile, label part). Each CTA sweeps one contiguous
// label range for one 128-query tile; all CTAs of a part stream the same W
// tiles at about the same time, so W comes from DRAM ~once per part and the
// other query tiles hit L2. Lists per query = n_parts * SPLIT.
struct Seg {
  int64_t qt, lt0, lt1;
  int slot;
};

__device__ __forceinline__ bool next_seg(int64_t& u, int64_t u1, const TcArgs& a, Seg& s) {
  if (u > u1) return false;  // exactly one (possibly empty) segment per CTA: empty ones flush zeros
  (void)a;
  s.qt = blockIdx.x;
  s.lt0 = u;
  s.lt1 = u1;
  s.slot = blockIdx.y;
  u = u1 + 1;
  return true;
}

// Scan one 32-column chunk of scores held in registers: a warp vote on the
// per-lane maxima skips the chunk unless some query can admit a candidate;
// candidates are appended (r[] indexed through a select tree, no local memory)
// and over-full buffers compacted once r[] is dead.
template <class Args>
__device__ __forceinline__ void scan_chunk(LaneTopK& tk, const uint32_t* r, int cn, uint32_t g0, bool active,
                                           const Args& a) {
  if (cn <= 0 || a.debug_no_topk) return;  // tile tail (uniform across the CTA)
  float t16[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float x0 = (j < cn) ? __uint_as_float(r[j]) : -INFINITY;
    const float x1 = (j + 16 < cn) ? __uint_as_float(r[j + 16]) : -INFINITY;
    t16[j] = fmaxf(x0, x1);
  }
#pragma unroll
  for (int w = 8; w > 0; w >>= 1)
#pragma unroll
    for (int j = 0; j < w; ++j) t16[j] = fmaxf(t16[j], t16[j + w]);
  if (a.dbg && (threadIdx.x & 31) == 0) atomicAdd(a.dbg + 3, 1ull);
  if (!__any_sync(0xffffffffu, active && t16[0] >= tk.tau_s)) return;  // the common case
  if (a.dbg && (threadIdx.x & 31) == 0) atomicAdd(a.dbg + 0, 1ull);
  uint32_t m = 0;
  if (active) {
#pragma unroll
    for (int j = 0; j < 32; ++j) m |= (j < cn && __uint_as_float(r[j]) >= tk.tau_s) ? (1u << j) : 0u;
  }
  while (m) {
    const int j = __ffs(m) - 1;
    m &= m - 1;
    lane_offer(tk, __uint_as_float(pick32(r, j)), g0 + j);
  }
  if (a.dbg) {
    const unsigned need = __ballot_sync(0xffffffffu, active && (tk.cnt - tk.nsorted) > a.cap / 2);
    if ((threadIdx.x & 31) == 0) atomicAdd(a.dbg + 2, static_cast<unsigned long long>(__popc(need)));
  }
  topk_settle(tk, a.cap, a.k, active);
}

// CL = cluster size along query tiles: the CL CTAs of a cluster sweep the same
// label tiles; each loads 1/CL of every W tile and multicasts it to all of them,
// so W leaves L2 once per cluster and the cluster moves in lockstep.
template <int SPLIT, int CL>
__global__ void __launch_bounds__(threads_for<SPLIT>(), 1)
    refresh_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs a) {
  constexpr int kEpiSplit = SPLIT;
  constexpr int kEpiWarps = 4 * SPLIT;
  constexpr uint16_t kMask = static_cast<uint16_t>((1u << CL) - 1);
  constexpr int B_SLICE = B_STAGE / CL;  // bytes of W tile rows loaded by each cluster rank
  const uint32_t crank = CL > 1 ? cluster_ctarank() : 0;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t u_begin = std::min<int64_t>(a.n_lt, static_cast<int64_t>(blockIdx.y) * a.tiles_per_part);
  const int64_t u_end = std::min<int64_t>(a.n_lt, u_begin + a.tiles_per_part);
  const int nkb = a.d / BK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // every cluster CTA's MMA must release the stage
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  if (CL > 1)
    cluster_sync_all();  // peers' barriers are initialised before any multicast targets them
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t u = u_begin;
      Seg sg;
      while (next_seg(u, u_end, a, sg)) {
        const int q0 = static_cast<int>(sg.qt * BM);
        for (int64_t t = sg.lt0; t < sg.lt1; ++t) {
          const int n0 = static_cast<int>(t * BN);
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], STAGE_BYTES);  // own A + all CL slices of the W tile
            tma_load_2d(sA + stage * A_STAGE, &tmA, &full[stage], kb * BK, q0);
            if (CL == 1)
              tma_load_2d(sB + stage * B_STAGE, &tmB, &full[stage], kb * BK, n0);
            else
              tma_load_2d_mc(sB + stage * B_STAGE + crank * B_SLICE, &tmB, &full[stage], kb * BK,
                             n0 + static_cast<int>(crank) * (BN / CL), kMask);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const int64_t n_units = u_end - u_begin;  // MMA tiles of this CTA, in schedule order
    for (int64_t t = 0; t < n_units; ++t) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t dcol = tmem_base + static_cast<uint32_t>(acc * BN);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint64_t ad = smem_desc(sA + stage * A_STAGE);
          const uint64_t bd = smem_desc(sB + stage * B_STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {
            // +32 B along K inside the 128 B swizzle atom = +2 in the encoded address
            mma_bf16(dcol, ad + 2 * kk, bd + 2 * kk, (kb | kk) != 0);
          }
          if (CL == 1)
            mma_commit(&empty[stage]);
          else
            mma_commit_mc(&empty[stage], kMask);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) mma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue: TMEM -> registers -> running top-k
    // warp e = warp - 4 reads TMEM lanes 32*(e%4).. (its lane quadrant, = warp % 4)
    // and columns [half*BN/2, (half+1)*BN/2) of every accumulator.
    const int e = warp - kEpiWarp0, quad = e & 3, half = e >> 2;
    const int row = quad * 32 + lane;  // TMEM lane = query row in tile
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    uint64_t* buf = a.bufs + ((static_cast<size_t>(blockIdx.x * gridDim.y + blockIdx.y) * kEpiSplit + half) * BM + row) *
                             (a.cap + kTopkSlack);
    constexpr int kCols = BN / kEpiSplit;
    int acc = 0;
    uint32_t acc_phase = 0;
    int64_t u = u_begin;
    Seg sg;
    while (next_seg(u, u_end, a, sg)) {
      const int64_t q = sg.qt * BM + row;
      const bool active = q < a.nq;
      LaneTopK tk;
      {
        const int64_t p0 = active ? a.pos_indptr[q] : 0, p1 = active ? a.pos_indptr[q + 1] : 0;
        lane_init(tk, buf, a.pos_ids + p0, p1 - p0, active ? a.gtau + q : nullptr);
      }
      uint64_t g_pref = 0;  // shared threshold prefetched one tile ahead
      for (int64_t t = sg.lt0; t < sg.lt1; ++t) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const int64_t n0 = t * BN;
        const int nvalid = static_cast<int>(std::min<int64_t>(BN, a.L - n0));
        // shared threshold: apply the value fetched during the previous tile, fetch the next
        if (tk.gtau) {
          if (g_pref > tk.tau) {
            tk.tau = g_pref;
            tk.tau_s = key_score(g_pref);
          }
          g_pref = *reinterpret_cast<volatile uint64_t*>(tk.gtau);
        }
        // 32-column chunks, the next chunk's TMEM load in flight while this one is scanned
        const uint32_t tbase = lane_base + static_cast<uint32_t>(acc * BN + half * kCols);
        const int col0 = half * kCols;
        uint32_t ra[32], rb[32];
        __syncwarp();
        tmem_ld32_nowait(tbase, ra);
        tmem_wait();
#pragma unroll 1
        for (int c = 0; c < kCols; c += 64) {
          __syncwarp();
          tmem_ld32_nowait(tbase + c + 32, rb);
          scan_chunk(tk, ra, nvalid - (col0 + c), static_cast<uint32_t>(n0 + col0 + c + a.off), active, a);
          __syncwarp();
          tmem_wait();
          __syncwarp();
          if (c + 64 < kCols) tmem_ld32_nowait(tbase + c + 64, ra);
          scan_chunk(tk, rb, nvalid - (col0 + c + 32), static_cast<uint32_t>(n0 + col0 + c + 32 + a.off), active, a);
          __syncwarp();
          tmem_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      const int list = sg.slot * kEpiSplit + half;
      uint64_t* out = a.part_keys + (static_cast<size_t>(list) * a.nq + (active ? q : 0)) * a.k;
      topk_flush(tk, a.cap, a.k, active, out);
    }
  }

  tc_fence_before();
  if (CL > 1)
    cluster_sync_all();  // no CTA leaves while peers may still signal its barriers
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

int make_map(CUtensorMap* m, const void* base, int64_t rows, int d, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return set_error(ASTRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ASTRA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return ASTRA_OK;
}

template <int SPLIT, int CL>
int launch_variant(const CUtensorMap& tmA, const CUtensorMap& tmB, const TcArgs& a, dim3 grid, cudaStream_t st) {
  static bool attr_set = false;
  auto kern = refresh_tc_kernel<SPLIT, CL>;
  if (!attr_set) {
    ASTRA_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(kSmemBytes)),
                         "smem attr"));
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads_for<SPLIT>());
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ASTRA_TRY(check_cuda(cudaLaunchKernelEx(&cfg, kern, tmA, tmB, a), "launch refresh_tc"));
  ASTRA_LAUNCHED("refresh_tc");
  return ASTRA_OK;
}

}  // namespace

// Cluster size along query tiles (ASTRA_TC_CLUSTER=1|2|4, default 2), reduced
// for batches with few query tiles.
int refresh_tc_cluster(int64_t n_qt) {
  static int cl = [] {
    const char* e = getenv("ASTRA_TC_CLUSTER");
    const int v = e ? atoi(e) : 2;
    return (v == 1 || v == 2 || v == 4) ? v : 2;
  }();
  int c = cl;
  while (c > 1 && n_qt < c) c >>= 1;
  return c;
}

// Epilogue split (ASTRA_TC_SPLIT=1|2, default 1: measured faster, fewer partial lists).
int refresh_tc_split() {
  static int split = [] {
    const char* e = getenv("ASTRA_TC_SPLIT");
    return (e && atoi(e) == 2) ? 2 : 1;
  }();
  return split;
}

// Number of CTAs and of partial lists per query for nq queries over L labels.
void refresh_tc_layout(int64_t nq, int64_t L, int* n_ctas, int* n_lists) {
  int64_t n_qt = std::max<int64_t>(1, (nq + BM - 1) / BM);
  const int cl = refresh_tc_cluster(n_qt);
  n_qt = (n_qt + cl - 1) / cl * cl;  // whole clusters (padding tiles hold no queries)
  const int64_t n_lt = std::max<int64_t>(1, (L + BN - 1) / BN);
  const int64_t parts = std::min<int64_t>(n_lt, std::max<int64_t>(1, num_sms() / n_qt));
  *n_ctas = static_cast<int>(n_qt * parts);
  *n_lists = static_cast<int>(parts) * refresh_tc_split();
}

int launch_refresh_tc(const uint16_t* qb, int64_t nq, int d, const uint16_t* wb, int64_t L, int64_t label_offset,
                      const int64_t* pos_indptr, const int32_t* pos_ids, int k, int cap, uint64_t* bufs,
                      uint64_t* part_keys, uint64_t* gtau, cudaStream_t st) {
  if ((reinterpret_cast<uintptr_t>(qb) & 15) || (reinterpret_cast<uintptr_t>(wb) & 15))
    return set_error(ASTRA_ERR_CONFIG, "bf16 operands must be 16-byte aligned");
  if (L <= 0) return ASTRA_OK;
  int G, n_lists;
  refresh_tc_layout(nq, L, &G, &n_lists);
  const int n_parts = n_lists / refresh_tc_split();
  const int cl = refresh_tc_cluster((nq + BM - 1) / BM);
  CUtensorMap tmA, tmB;
  ASTRA_TRY(make_map(&tmA, qb, nq, d, BM));
  ASTRA_TRY(make_map(&tmB, wb, L, d, BN / cl));
  TcArgs a;
  a.nq = nq;
  a.L = L;
  a.off = label_offset;
  a.d = d;
  a.k = k;
  a.cap = cap;
  a.n_lt = (L + BN - 1) / BN;
  a.tiles_per_part = (a.n_lt + n_parts - 1) / n_parts;
  a.pos_indptr = pos_indptr;
  a.pos_ids = pos_ids;
  a.bufs = bufs;
  a.part_keys = part_keys;
  a.gtau = gtau;
  a.debug_no_topk = getenv("ASTRA_TC_DEBUG_NO_TOPK") != nullptr;
  static unsigned long long* dbg_buf = nullptr;
  const bool counters = getenv("ASTRA_TC_DEBUG_COUNTERS") != nullptr;
  if (counters && !dbg_buf) cudaMalloc(&dbg_buf, 4 * sizeof(unsigned long long));
  a.dbg = counters ? dbg_buf : nullptr;
  if (counters) cudaMemsetAsync(dbg_buf, 0, 4 * sizeof(unsigned long long), st);
  ASTRA_TRY(check_cuda(cudaMemsetAsync(gtau, 0, sizeof(uint64_t) * nq, st), "memset gtau"));
  const dim3 grid(static_cast<unsigned>(G / n_parts), static_cast<unsigned>(n_parts));
  const int split = refresh_tc_split();
  if (counters) {
    int rc = split == 1 ? (cl == 2 ? launch_variant<1, 2>(tmA, tmB, a, grid, st) : launch_variant<1, 1>(tmA, tmB, a, grid, st))
                        : launch_variant<2, 1>(tmA, tmB, a, grid, st);
    unsigned long long h[4];
    cudaMemcpyAsync(h, dbg_buf, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[refresh_tc] nq=%lld k=%d slow_chunks=%llu/%llu (%.3f) cnt_sum_at_settle=%llu compactions=%llu\n",
            (long long)nq, k, h[0], h[3], h[3] ? double(h[0]) / h[3] : 0.0, h[1], h[2]);
    return rc;
  }
  if (split == 1 && cl == 1) return launch_variant<1, 1>(tmA, tmB, a, grid, st);
  if (split == 1 && cl == 2) return launch_variant<1, 2>(tmA, tmB, a, grid, st);
  if (split == 1 && cl == 4) return launch_variant<1, 4>(tmA, tmB, a, grid, st);
  if (split == 2 && cl == 1) return launch_variant<2, 1>(tmA, tmB, a, grid, st);
  if (split == 2 && cl == 2) return launch_variant<2, 2>(tmA, tmB, a, grid, st);
  return launch_variant<2, 4>(tmA, tmB, a, grid, st);
}

}  // namespace astra
