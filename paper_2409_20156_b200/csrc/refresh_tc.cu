// refresh_tc.cu — bf16 / e4m3 tcgen05 GEMM of queries x labels with a fused
// top-k epilogue: the B200 shortlist refresh (replaces anns.py:253-256).
// The e4m3 instance (kind::f8f6f4) runs the same pipeline on 8-bit operands:
// identical 128-byte swizzle rows carrying twice the K extent per stage.
//
// One CTA owns a 128-query tile and sweeps a contiguous range of label tiles
// (N = 256 labels each). Warp roles (256 threads):
//   warp 0      TMA producer: A (128 x 64 bf16) and B (256 x 64 bf16) k-blocks,
//               SWIZZLE_128B, into a 4-stage shared-memory ring (48 KB/stage);
//               with a cluster of CL query tiles each CTA loads 1/CL of every
//               W tile and multicasts it to the cluster.
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.kind::f16
//               (M=128, N=256, K=16) into a TMEM accumulator; tcgen05.commit
//               releases smem stages and publishes finished accumulators.
//               Default: CTA pairs (cta_group::2): the even CTA of a cluster
//               of 2 issues M=256 MMAs over both CTAs' shared memory (each
//               stages its 128 query rows and 128 of the tile's 256 W rows,
//               6 x 32 KB ring), commits to both CTAs' barriers.
//   warp 2      TMEM allocator (512 columns = 2 accumulators of 256 fp32 cols).
//   warps 4-7   epilogue: tcgen05.ld 64 columns per step (thread = query row =
//               TMEM lane), one warp vote per step, then either
//                 RUNNING  exact running top-k per query (topk.cuh), or
//                 FIXED    append every key >= a per-query threshold to a
//                          candidate list (no compaction, no bursts), or
//                 GMAX     write the maximum of every 64-label group (the
//                          sample pass: a threshold source).
// Scores never leave the SM. refresh.cu composes the two modes into the
// sample / threshold / select / verify pipeline (see the comment there).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"
#include "refresh_tc.cuh"
#include "topk.cuh"

namespace astra {
namespace {

constexpr int BM = 128, BN = kTcTileLabels, BK = 64, UMMA_K = 16, STAGES = 4;
constexpr int A_STAGE = BM * BK * 2;  // 16 KB
constexpr int B_STAGE = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
constexpr int TMEM_COLS = 512;
constexpr int kEpiWarp0 = 4, kEpiWarps = 4;
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);
constexpr size_t kBarrierBytes = 1024;  // mbarriers, TMEM address, only_flagged bitmap
constexpr int kQtBits = 6144;           // query-tile clusters covered by the bitmap
// + one 256 B score-staging row per epilogue thread (slow path of scan64)
constexpr size_t kSmemBytes = 1024 /*align slack*/ + STAGES * STAGE_BYTES + kBarrierBytes + kEpiWarps * 32 * 256;

// idesc for kind::f16: D=F32, A=B=BF16, both K-major, N>>3 at [17,23), M>>4 at [24,29)
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
// CTA pair (cta_group::2): M = 256 (128 query rows per CTA), N = 256 (each CTA holds 128 W rows)
constexpr uint32_t kIdescPair =
    (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t((2 * BM) >> 4) << 24);

// idesc for kind::f8f6f4: D=F32, A=B=E4M3 (format 0 at [7,10) and [10,13)), both K-major
constexpr uint32_t kIdescF8 = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
constexpr uint32_t kIdescPairF8 = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t((2 * BM) >> 4) << 24);
// K elements per 128-byte swizzle row: 64 bf16 or 128 e4m3. Each MMA consumes
// 32 bytes of K (16 bf16 / 32 e4m3), so a stage holds BK / UMMA_K = 4 MMAs
// either way and the shared-memory layout is identical; an e4m3 stage carries
// twice the K extent (and twice the flops) of a bf16 one.
template <bool F8>
constexpr int kb_elems() { return F8 ? 2 * BK : BK; }

// Shared-memory ring geometry: single CTA (4 x 48 KB: A 128 rows + B 256 rows)
// or CTA pair (6 x 32 KB: A 128 rows + this CTA's 128 of the 256 B rows).
template <bool PAIR>
struct Geo {
  static constexpr int B_ROWS = PAIR ? BN / 2 : BN;
  static constexpr int B_ST = B_ROWS * BK * 2;
  static constexpr int STG = A_STAGE + B_ST;
  static constexpr int NST = PAIR ? 6 : STAGES;
};

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

__device__ __forceinline__ void mma_f8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescF8), "r"(accumulate));
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

// Pair TMA load: lands in this CTA's smem, completes tx on the LEADER's barrier
// (bar_cluster = its shared::cluster address).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

// shared::cluster address of `p` (a shared::cta address) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_cluster(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

// Relaxed remote arrive (no MEMBAR.GPU: a release here made every epilogue
// warp wait for its outstanding candidate stores once per tile). Only the
// TMEM reads must precede the arrive, and tcgen05.wait::ld has completed them
// (ordered by tcgen05.fence::before_thread_sync) before it is issued.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
#ifdef ASTRA_TC_RELEASE_ARRIVE  // (A/B switch: the release form)
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
#else
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
#endif
}

__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescPair), "r"(accumulate));
}

__device__ __forceinline__ void mma_f8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescPairF8), "r"(accumulate));
}

// Arrive on `bar` in every CTA of `mask` (the pair, or every pair sharing the
// stage's W rows) once the leader's prior tcgen05.mma complete.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
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

struct TcArgs {
  int64_t nq, L, off;
  int d, k, cap;
  int64_t n_lt, tiles_per_part, tile_stride;  // swept label tiles, per part, stride between them
  int64_t n_qt_cl;                            // query-tile clusters (CL query tiles each)
  int n_parts;                                // label parts (= partial lists per query)
  const int64_t* pos_indptr;
  const int32_t* pos_ids;
  uint64_t* bufs;       // RUNNING: per-lane buffers
  uint64_t* part_keys;  // RUNNING: [n_parts][nq][k]
  uint64_t* gtau;       // RUNNING: nq shared thresholds (zeroed by the host before launch)
  const uint64_t* tau_in;  // FIXED: threshold of query q = tau_in[q * tau_stride]
  int tau_stride;
  uint64_t* cand;          // FIXED: [n_parts][nq][cand_cap]
  int32_t* cand_cnt;       // FIXED: [n_parts][nq]
  int cand_cap;
  uint32_t* gmax;          // GMAX: [nq][n_lt * 4] orderable bits of the 64-label group maxima
  const int32_t* only_flagged;
  // compact verify (running mode): rows are the flagged queries gathered in
  // front (*n_active of them); qmap[row] = the original query (positives)
  const int32_t* qmap;
  const int32_t* n_active;
  int debug_no_topk;  // ASTRA_TC_DEBUG_NO_TOPK=1: skip selection (pipeline-rate measurement only)
  // ASTRA_TC_DEBUG_COUNTERS=1: [slow steps, -, compactions, steps, then clock64 cycle sums:
  // 4 epi tfull wait, 5 epi fast path, 6 epi slow path, 7 epi settle, 8 epi total,
  // 9 mma tempty wait, 10 mma full wait, 11 mma total]
  unsigned long long* dbg;
};

enum { kRunning = 0, kFixed = 1, kGmax = 2 };

struct EpiProf {
  long long fast = 0, slow = 0, settle = 0;
};

// Admit one score (RUNNING: key > tau into the lane buffer, room guaranteed by
// topk_settle; FIXED: key >= tau into the candidate list, counting past the
// capacity — overflow is detected by the select pass).
template <bool FIXED>
__device__ __forceinline__ void admit(LaneTopK& tk, float s, uint32_t gid, int cand_cap) {
  if (s >= tk.tau_s) {
    if constexpr (FIXED) {
      const uint64_t key = make_key(s, gid);
      if (key >= tk.tau) {
        if (tk.cnt < cand_cap) tk.buf[tk.cnt] = key;
        ++tk.cnt;
      }
    } else {
      lane_offer(tk, s, gid);
    }
  }
}

// Scan 64 columns held in registers (ra = columns 0-31, rb = 32-63 of the
// step). Fast path: an FMNMX3 max tree over the 64 scores and ONE warp vote;
// the warp skips the step unless some query can admit a candidate. Slow path:
// the tree level with 8 maxima (group g = columns g + 8i) picks the groups to
// inspect; the step is staged in the lane's 256 B shared-memory row with group
// g's 8 scores in 16 B chunks 2g, 2g+1 (chunk c stored at c ^ (lane & 7):
// conflict-free STS.128), so a flagged group costs two LDS.128 and 8 compares.
// The tile-tail guards exist only in the !FULL instance.
template <bool FULL, bool FIXED, class Args>
__device__ __forceinline__ void scan64(LaneTopK& tk, const uint32_t* ra, const uint32_t* rb, int cn, uint32_t g0,
                                       bool active, const Args& a, float* stage, EpiProf& pf) {
  if (!FULL && cn <= 0) return;  // tile tail (uniform across the CTA)
  if (a.debug_no_topk) return;
  const long long c0 = a.dbg ? clock64() : 0;
  auto val = [&](int col) -> float {  // score of column col (compile-time) of the step, -inf past the tail
    const float v = __uint_as_float(col < 32 ? ra[col] : rb[col - 32]);
    return (FULL || col < cn) ? v : -INFINITY;
  };
  float t[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) t[j] = fmaxf(val(j), val(j + 32));
#pragma unroll
  for (int j = 0; j < 16; ++j) t[j] = fmaxf(t[j], t[j + 16]);
  float grp[8];  // grp[g] = max of columns g + 8i, i < 8
#pragma unroll
  for (int j = 0; j < 8; ++j) grp[j] = fmaxf(t[j], t[j + 8]);
  const float m = fmaxf(fmaxf(fmaxf(grp[0], grp[1]), fmaxf(grp[2], grp[3])),
                        fmaxf(fmaxf(grp[4], grp[5]), fmaxf(grp[6], grp[7])));
  const bool want = active && m >= tk.tau_s;
  const bool any = __any_sync(0xffffffffu, want);
  if (a.dbg && (threadIdx.x & 31) == 0) atomicAdd(a.dbg + 3, 1ull);
  const long long c1 = a.dbg ? clock64() : 0;
  if (a.dbg) pf.fast += c1 - c0;
  if (!any) return;
  if (a.dbg && (threadIdx.x & 31) == 0) atomicAdd(a.dbg + 0, 1ull);
  const int sw = threadIdx.x & 7;
  uint32_t gm = 0;
  if (want) {
#pragma unroll
    for (int g = 0; g < 8; ++g) gm |= grp[g] >= tk.tau_s ? (1u << g) : 0u;
  }
  // stage only the flagged groups (predicated stores: shared-memory traffic
  // proportional to the lanes that have candidates)
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    if (gm & (1u << g)) {
      *reinterpret_cast<float4*>(stage + (((2 * g) ^ sw) << 2)) =
          make_float4(val(g), val(g + 8), val(g + 16), val(g + 24));
      *reinterpret_cast<float4*>(stage + (((2 * g + 1) ^ sw) << 2)) =
          make_float4(val(g + 32), val(g + 40), val(g + 48), val(g + 56));
    }
  }
  while (gm) {
    const int g = __ffs(gm) - 1;
    gm &= gm - 1;
    const float4 x = *reinterpret_cast<const float4*>(stage + (((2 * g) ^ sw) << 2));
    const float4 y = *reinterpret_cast<const float4*>(stage + (((2 * g + 1) ^ sw) << 2));
    const uint32_t gg = g0 + g;
    admit<FIXED>(tk, x.x, gg, a.cand_cap);
    admit<FIXED>(tk, x.y, gg + 8, a.cand_cap);
    admit<FIXED>(tk, x.z, gg + 16, a.cand_cap);
    admit<FIXED>(tk, x.w, gg + 24, a.cand_cap);
    admit<FIXED>(tk, y.x, gg + 32, a.cand_cap);
    admit<FIXED>(tk, y.y, gg + 40, a.cand_cap);
    admit<FIXED>(tk, y.z, gg + 48, a.cand_cap);
    admit<FIXED>(tk, y.w, gg + 56, a.cand_cap);
  }
  __syncwarp();
  if constexpr (!FIXED) {
    long long c2 = 0;
    if (a.dbg) {
      const unsigned need = __ballot_sync(0xffffffffu, active && (tk.cnt - tk.nsorted) > a.cap / 2);
      if ((threadIdx.x & 31) == 0) atomicAdd(a.dbg + 2, static_cast<unsigned long long>(__popc(need)));
      c2 = clock64();
      pf.slow += c2 - c1;
    }
    topk_settle(tk, a.cap, a.k, active);  // <= 64 appends per lane since the last settle (kTopkSlack)
    if (a.dbg) pf.settle += clock64() - c2;
  } else {
    if (a.dbg) pf.slow += clock64() - c1;
  }
}

// One work unit = (cluster of CL query tiles, label part): the CL CTAs of a
// cluster sweep the same contiguous range of swept label tiles; each loads
// 1/CL of every W tile and multicasts it to all of them. Clusters are
// persistent: cluster c takes units c, c + n_clusters, ... (unit uc = part *
// n_qt_cl + query-tile cluster), so the grid can be sized to an SM budget and
// the query tiles of a part stream the same W tiles at about the same time (W
// comes from DRAM ~once per part; the other query tiles hit L2).
struct Unit {
  int64_t qt;      // this CTA's query tile
  int part;        // label part = the query's partial list index
  int64_t t0, t1;  // swept label tiles [t0, t1)
};

template <int CL>
__device__ __forceinline__ Unit unit_of(const TcArgs& a, int64_t n_qt_cl, int64_t uc, uint32_t crank) {
  Unit u;
  const int64_t qc = uc % n_qt_cl;
  u.part = static_cast<int>(uc / n_qt_cl);
  u.qt = qc * CL + crank;
  u.t0 = std::min<int64_t>(a.n_lt, static_cast<int64_t>(u.part) * a.tiles_per_part);
  u.t1 = std::min<int64_t>(a.n_lt, u.t0 + a.tiles_per_part);
  return u;
}

// only_flagged: 1 bit per query-tile cluster in shared memory (all roles skip
// the same units); clusters beyond the bitmap are always active.
__device__ __forceinline__ bool unit_active(const uint32_t* qbits, int64_t n_qt_cl, int64_t uc) {
  if (!qbits) return true;
  const int64_t qc = uc % n_qt_cl;
  if (qc >= kQtBits) return true;
  return (qbits[qc >> 5] >> (qc & 31)) & 1u;
}

template <int CL, int MODE, bool PAIR, bool F8>
__global__ void __launch_bounds__(kThreads, 1)
    refresh_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcArgs a) {
  // (two CTA pairs per cluster sharing every W tile by multicast were measured
  // 1.7x slower: profiles/r02s3/ab_refresh_cluster4.txt)
  static_assert(!PAIR || CL == 2, "a CTA pair is a cluster of 2");
  using G = Geo<PAIR>;
  constexpr int NST = G::NST;
  constexpr uint16_t kMask = static_cast<uint16_t>((1u << CL) - 1);
  constexpr int B_SLICE = B_STAGE / CL;  // bytes of W tile rows loaded by each cluster rank (multicast)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = CL > 1 ? cluster_ctarank() : 0;
  const int64_t cluster = blockIdx.x / CL, n_clusters = gridDim.x / CL;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;
  unsigned char* sB = smem + NST * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * G::STG);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* qbits_s = tmem_holder + 8;  // kQtBits bits
  float* stage_base = reinterpret_cast<float*>(smem + NST * G::STG + kBarrierBytes);
  const bool leader = !PAIR || (crank & 1u) == 0;
  const uint32_t prank = crank & ~1u;  // this CTA's pair leader
  const uint16_t pair_mask = static_cast<uint16_t>(3u << prank);
  constexpr int KB = kb_elems<F8>();  // K elements per stage
  const int nkb = a.d / KB;
  // query rows in play: all nq, or (compact verify) the *n_active gathered ones
  const int64_t nq_eff = a.n_active ? static_cast<int64_t>(*a.n_active) : a.nq;
  const int64_t n_qt_cl = a.n_active ? (nq_eff + CL * BM - 1) / (CL * BM) : a.n_qt_cl;
  const int64_t n_units = n_qt_cl * a.n_parts;

  const uint32_t* qbits = nullptr;
  if (a.only_flagged) {
    // verification fallback: which query-tile clusters hold a flagged query
    for (int i = threadIdx.x; i < kQtBits / 32; i += kThreads) qbits_s[i] = 0u;
    __syncthreads();
    const int64_t nq_bits = std::min<int64_t>(a.nq, static_cast<int64_t>(kQtBits) * CL * BM);
    for (int64_t q = threadIdx.x; q < nq_bits; q += kThreads)
      if (a.only_flagged[q]) {
        const int64_t qc = q / (CL * BM);
        atomicOr(&qbits_s[qc >> 5], 1u << (qc & 31));
      }
    qbits = qbits_s;
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      // multicast: every cluster CTA's MMA releases the stage; pair: one commit from the leader
      mbar_init(&empty[s], PAIR ? 1 : CL);  // multicast: every cluster CTA's MMA releases the stage; pair: the leader's commit
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], PAIR ? 2 * kEpiWarps : kEpiWarps);  // pair: both CTAs' epilogues free the leader's MMA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
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
      for (int64_t uc = cluster; uc < n_units; uc += n_clusters) {
        if (!unit_active(qbits, n_qt_cl, uc)) continue;
        const Unit un = unit_of<CL>(a, n_qt_cl, uc, crank);
        const int q0 = static_cast<int>(un.qt * BM);
        for (int64_t t = un.t0; t < un.t1; ++t) {
          const int n0 = static_cast<int>(t * a.tile_stride * BN);
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            if constexpr (PAIR) {
              // both CTAs load their A rows and their half of the W tile; the
              // transaction bytes of both complete on the leader's barrier
              const uint32_t bar = mapa_cluster(&full[stage], prank);
              if (leader) mbar_expect_tx(&full[stage], 2 * G::STG);
              tma_load_2d_pair(sA + stage * A_STAGE, &tmA, bar, kb * KB, q0);
              tma_load_2d_pair(sB + stage * G::B_ST, &tmB, bar, kb * KB, n0 + static_cast<int>(crank) * G::B_ROWS);
            } else {
              mbar_expect_tx(&full[stage], STAGE_BYTES);  // own A + all CL slices of the W tile
              tma_load_2d(sA + stage * A_STAGE, &tmA, &full[stage], kb * KB, q0);
              if (CL == 1)
                tma_load_2d(sB + stage * B_STAGE, &tmB, &full[stage], kb * KB, n0);
              else
                tma_load_2d_mc(sB + stage * B_STAGE + crank * B_SLICE, &tmB, &full[stage], kb * KB,
                               n0 + static_cast<int>(crank) * (BN / CL), kMask);
            }
            if (++stage == NST) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (pair: the leader CTA issues for both)
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    long long p_te = 0, p_full = 0;
    const long long p_t0 = a.dbg ? clock64() : 0;
    for (int64_t uc = cluster; uc < n_units; uc += n_clusters) {
      if (!unit_active(qbits, n_qt_cl, uc)) continue;
      const Unit un = unit_of<CL>(a, n_qt_cl, uc, crank);
      for (int64_t t = un.t0; t < un.t1; ++t) {
        long long w0 = a.dbg ? clock64() : 0;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        if (a.dbg) p_te += clock64() - w0;
        tc_fence_after();
        const uint32_t dcol = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < nkb; ++kb) {
          w0 = a.dbg ? clock64() : 0;
          mbar_wait(&full[stage], phase);
          if (a.dbg) p_full += clock64() - w0;
          tc_fence_after();
          if (lane == 0) {
            const uint64_t ad = smem_desc(sA + stage * A_STAGE);
            const uint64_t bd = smem_desc(sB + stage * G::B_ST);
#pragma unroll
            for (int kk = 0; kk < BK / UMMA_K; ++kk) {
              // +32 B along K inside the 128 B swizzle atom = +2 in the encoded address
              if constexpr (PAIR && F8)
                mma_f8_pair(dcol, ad + 2 * kk, bd + 2 * kk, (kb | kk) != 0);
              else if constexpr (PAIR)
                mma_bf16_pair(dcol, ad + 2 * kk, bd + 2 * kk, (kb | kk) != 0);
              else if constexpr (F8)
                mma_f8(dcol, ad + 2 * kk, bd + 2 * kk, (kb | kk) != 0);
              else
                mma_bf16(dcol, ad + 2 * kk, bd + 2 * kk, (kb | kk) != 0);
            }
            if constexpr (PAIR)
              mma_commit_pair(&empty[stage], pair_mask);
            else if (CL == 1)
              mma_commit(&empty[stage]);
            else
              mma_commit_mc(&empty[stage], kMask);
          }
          __syncwarp();
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) {
          if constexpr (PAIR)
            mma_commit_pair(&tfull[acc], pair_mask);
          else
            mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    if (a.dbg && lane == 0) {
      atomicAdd(a.dbg + 9, static_cast<unsigned long long>(p_te));
      atomicAdd(a.dbg + 10, static_cast<unsigned long long>(p_full));
      atomicAdd(a.dbg + 11, static_cast<unsigned long long>(clock64() - p_t0));
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue: TMEM -> registers -> per-query selection
    // warp e = warp - 4 reads TMEM lanes 32*e.. (its lane quadrant, = warp % 4)
    const int e = warp - kEpiWarp0;
    const int row = e * 32 + lane;  // TMEM lane = query row in tile
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(e * 32) << 16);
    float* stage = stage_base + (e * 32 + lane) * 64;
    uint64_t* const run_buf = a.bufs ? a.bufs + (static_cast<size_t>(blockIdx.x) * BM + row) * (a.cap + kTopkSlack)
                                     : nullptr;
    int acc = 0;
    uint32_t acc_phase = 0;
    EpiProf pf;
    long long p_wait = 0;
    const long long p_t0 = a.dbg ? clock64() : 0;
    for (int64_t uc = cluster; uc < n_units; uc += n_clusters) {
      if (!unit_active(qbits, n_qt_cl, uc)) continue;
      const Unit un = unit_of<CL>(a, n_qt_cl, uc, crank);
      const int64_t q = un.qt * BM + row;
      const bool active = q < nq_eff;
      const int list = un.part;
      LaneTopK tk;
      if constexpr (MODE == kGmax) {
        lane_init(tk, nullptr, nullptr, 0);
      } else if constexpr (MODE == kFixed) {
        lane_init(tk, a.cand + (static_cast<size_t>(list) * a.nq + (active ? q : 0)) * a.cand_cap, nullptr, 0);
        tk.tau = active ? a.tau_in[static_cast<size_t>(q) * a.tau_stride] : ~0ull;
        tk.tau_s = tk.tau ? key_score(tk.tau) : -INFINITY;
      } else {
        const int64_t qo = active && a.qmap ? static_cast<int64_t>(a.qmap[q]) : q;  // positives of the original query
        const int64_t p0 = active ? a.pos_indptr[qo] : 0, p1 = active ? a.pos_indptr[qo + 1] : 0;
        lane_init(tk, run_buf, a.pos_ids + p0, p1 - p0, active ? a.gtau + q : nullptr);
      }
      uint64_t g_pref = 0;  // RUNNING: shared threshold prefetched one tile ahead
      for (int64_t t = un.t0; t < un.t1; ++t) {
        const long long w0 = a.dbg ? clock64() : 0;
        mbar_wait(&tfull[acc], acc_phase);
        if (a.dbg) p_wait += clock64() - w0;
        tc_fence_after();
        const int64_t n0 = t * a.tile_stride * BN;
        const int nvalid = static_cast<int>(std::min<int64_t>(BN, a.L - n0));
        if constexpr (MODE == kRunning) {
          // shared threshold: apply the value fetched during the previous tile, fetch the next
          if (tk.gtau) {
            if (g_pref > tk.tau) {
              tk.tau = g_pref;
              tk.tau_s = key_score(g_pref);
            }
            g_pref = *reinterpret_cast<volatile uint64_t*>(tk.gtau);
          }
        }
        // 64-column steps: two 32-column TMEM loads, one wait, one vote
        const uint32_t tbase = lane_base + static_cast<uint32_t>(acc * BN);
        const bool full_tile = nvalid == BN;
        if constexpr (MODE == kGmax) {
          uint32_t gm[4];
#pragma unroll
          for (int c = 0; c < BN; c += 64) {
            uint32_t ra[32], rb[32];
            __syncwarp();
            tmem_ld32_nowait(tbase + c, ra);
            tmem_ld32_nowait(tbase + c + 32, rb);
            tmem_wait();
            float m = -INFINITY;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float x0 = (full_tile || c + j < nvalid) ? __uint_as_float(ra[j]) : -INFINITY;
              const float x1 = (full_tile || c + j + 32 < nvalid) ? __uint_as_float(rb[j]) : -INFINITY;
              m = fmaxf(m, fmaxf(x0, x1));
            }
            gm[c / 64] = ord_bits(__float_as_uint(__fadd_rn(m, 0.0f)));  // -inf: empty group, below every score
          }
          if (active)
            *reinterpret_cast<uint4*>(a.gmax + static_cast<size_t>(q) * (a.n_lt * 4) + t * 4) =
                make_uint4(gm[0], gm[1], gm[2], gm[3]);
        } else {
#pragma unroll 1
          for (int c = 0; c < BN; c += 64) {
            uint32_t ra[32], rb[32];
            __syncwarp();
            tmem_ld32_nowait(tbase + c, ra);
            tmem_ld32_nowait(tbase + c + 32, rb);
            tmem_wait();
            const uint32_t g0 = static_cast<uint32_t>(n0 + c + a.off);
            if (full_tile)
              scan64<true, MODE == kFixed>(tk, ra, rb, 64, g0, active, a, stage, pf);
            else
              scan64<false, MODE == kFixed>(tk, ra, rb, nvalid - c, g0, active, a, stage, pf);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR)
            mbar_arrive_cluster(mapa_cluster(&tempty[acc], prank));  // the leader's MMA reuses both halves
          else
            mbar_arrive(&tempty[acc]);
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if constexpr (MODE == kFixed) {
        if (active) a.cand_cnt[static_cast<size_t>(list) * a.nq + q] = tk.cnt;
      } else if constexpr (MODE == kRunning) {
        uint64_t* out = a.part_keys + (static_cast<size_t>(list) * a.nq + (active ? q : 0)) * a.k;
        topk_flush(tk, a.cap, a.k, active, out);
      }
    }
    if (a.dbg && lane == 0) {
      atomicAdd(a.dbg + 4, static_cast<unsigned long long>(p_wait));
      atomicAdd(a.dbg + 5, static_cast<unsigned long long>(pf.fast));
      atomicAdd(a.dbg + 6, static_cast<unsigned long long>(pf.slow));
      atomicAdd(a.dbg + 7, static_cast<unsigned long long>(pf.settle));
      atomicAdd(a.dbg + 8, static_cast<unsigned long long>(clock64() - p_t0));
    }
  }

  tc_fence_before();
  if (CL > 1)
    cluster_sync_all();  // no CTA leaves while peers may still signal its barriers
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    else
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

// 2-D K-major map of a [rows, d] operand: bf16 (box 64 x box_rows) or e4m3
// bytes (box 128 x box_rows): 128-byte rows either way, SWIZZLE_128B.
int make_map(CUtensorMap* m, const void* base, int64_t rows, int d, int box_rows, bool f8) {
  auto fn = encode_fn();
  if (!fn) return set_error(ASTRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * (f8 ? 1 : 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(f8 ? 2 * BK : BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, f8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                  dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ASTRA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return ASTRA_OK;
}

template <int CL, int MODE, bool PAIR, bool F8>
int launch_variant(const CUtensorMap& tmA, const CUtensorMap& tmB, const TcArgs& a, dim3 grid, cudaStream_t st) {
  static bool attr_set = false;
  auto kern = refresh_tc_kernel<CL, MODE, PAIR, F8>;
  if (!attr_set) {
    ASTRA_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(kSmemBytes)),
                         "smem attr"));
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
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

bool refresh_tc_pair() {
  static const bool pair = [] {
    const char* e = getenv("ASTRA_TC_PAIR");
    return !(e && atoi(e) == 0);
  }();
  return pair;
}

// Cluster size along query tiles (ASTRA_TC_CLUSTER=1|2, default 2), reduced
// for batches with a single query tile.
int refresh_tc_cluster(int64_t n_qt) {
  static int cl = [] {
    const char* e = getenv("ASTRA_TC_CLUSTER");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  int c = cl;
  while (c > 1 && n_qt < c) c >>= 1;
  return c;
}

}  // namespace

static std::atomic<int> g_refresh_sm_budget{0};

void set_refresh_sm_budget(int n_sms) { g_refresh_sm_budget.store(n_sms > 0 ? n_sms : 0); }

// Persistent grid: at most one CTA per SM of the budget (astra_set_refresh_sm_budget,
// default every SM); the fewest label parts whose (query-tile cluster, part)
// units keep >= 93% of the budget's clusters busy over whole rounds.
void refresh_tc_layout(int64_t nq, int64_t n_tiles, int* n_ctas, int* n_parts) {
  const int64_t n_qt = std::max<int64_t>(1, (nq + BM - 1) / BM);
  const int cl = refresh_tc_cluster(n_qt);
  const int64_t n_qt_cl = (n_qt + cl - 1) / cl;
  n_tiles = std::max<int64_t>(1, n_tiles);
  int budget = num_sms();
  const int b = g_refresh_sm_budget.load();
  if (b > 0) budget = std::min(budget, b);
  const int64_t n_cl_max = std::max(1, budget / cl);
  // efficiency of p parts: useful unit-rounds / (rounds x clusters), counted in
  // label tiles (the last part of a query tile may be shorter)
  auto eff_of = [&](int64_t p) {
    const int64_t units = n_qt_cl * p;
    const int64_t n_cl = std::min(n_cl_max, units);
    const int64_t rounds = (units + n_cl - 1) / n_cl;
    const int64_t tpp = (n_tiles + p - 1) / p;
    return static_cast<double>(units) / static_cast<double>(rounds * n_cl_max) *
           static_cast<double>(n_tiles) / static_cast<double>(tpp * p);
  };
  // fewest parts that fill the budget (fewer lists, more L2 reuse of W): the
  // fewest reaching 93% (C4: 2 parts x 36 query-tile pairs on 144 SMs, W read
  // from DRAM once); with `fill`, a layout keeping every cluster busy to
  // within 1% (e.g. 37 parts x 36 pairs = 18 rounds of 74 pairs) while parts
  // stay >= 64 tiles long
  // ASTRA_REFRESH_FILL=1: prefer a layout that fills every SM pair to within
  // 1% (at C4: 37 parts on 148 SMs). Off by default: its units of one part
  // start in different rounds, so W is read ~1.5x from DRAM instead of once;
  // same-box A/B (profiles/r02s3/ab_refresh_fill2.txt): threshold pass 1.2%
  // faster at C4, but 2.6% slower at the C5 shard, whose 72 ms pass runs at
  // the power cap (the extra DRAM traffic lowers the clock).
  static const bool fill = [] {
    const char* e = getenv("ASTRA_REFRESH_FILL");
    return e && atoi(e) == 1;
  }();
  int64_t best_p = 1;
  double best_eff = -1.0;
  const int64_t p_max = std::min<int64_t>(n_tiles, 64);
  for (int64_t p = 1; p <= (fill ? p_max : 0); ++p) {
    if (p > 1 && n_tiles / p < 64) break;
    if (eff_of(p) >= 0.99) {
      best_p = p;
      best_eff = eff_of(p);
      break;
    }
  }
  if (best_eff < 0.0) {
    for (int64_t p = 1; p <= p_max; ++p) {
      const double eff = eff_of(p);
      if (eff > best_eff + 0.02) {
        best_eff = eff;
        best_p = p;
      }
      if (best_eff >= 0.93) break;
    }
  }
  *n_ctas = static_cast<int>(std::min(n_cl_max, n_qt_cl * best_p) * cl);
  *n_parts = static_cast<int>(best_p);
}

int launch_refresh_tc(const TcLaunch& p, cudaStream_t st) {
  if ((reinterpret_cast<uintptr_t>(p.qb) & 15) || (reinterpret_cast<uintptr_t>(p.wb) & 15))
    return set_error(ASTRA_ERR_CONFIG, "tensor-core operands must be 16-byte aligned");
  if (p.f8 && p.d % (2 * BK)) return set_error(ASTRA_ERR_CONFIG, "e4m3 refresh needs d %% 128 == 0 (d=%d)", p.d);
  if (p.L <= 0 || p.nq <= 0) return ASTRA_OK;
  const int64_t n_tiles_all = (p.L + BN - 1) / BN;
  const int64_t n_lt = (n_tiles_all + p.tile_stride - 1) / p.tile_stride;
  int G, n_parts;
  refresh_tc_layout(p.nq, n_lt, &G, &n_parts);
  const int cl = refresh_tc_cluster((p.nq + BM - 1) / BM);
  if (p.n_parts_fixed > 0) {  // compact verify: row count known on the device only
    n_parts = static_cast<int>(std::min<int64_t>(p.n_parts_fixed, n_lt));
    int budget = num_sms();
    const int b = g_refresh_sm_budget.load();
    if (b > 0) budget = std::min(budget, b);
    G = std::max(1, budget / cl) * cl;
  }
  CUtensorMap tmA, tmB;
  ASTRA_TRY(make_map(&tmA, p.qb, p.nq, p.d, BM, p.f8));
  ASTRA_TRY(make_map(&tmB, p.wb, p.L, p.d, BN / cl, p.f8));
  TcArgs a;
  a.nq = p.nq;
  a.L = p.L;
  a.off = p.off;
  a.d = p.d;
  a.k = p.k;
  a.cap = p.cap;
  a.n_lt = n_lt;
  a.tiles_per_part = (n_lt + n_parts - 1) / n_parts;
  a.tile_stride = p.tile_stride;
  a.n_qt_cl = ((p.nq + BM - 1) / BM + cl - 1) / cl;
  a.n_parts = n_parts;
  a.pos_indptr = p.pos_indptr;
  a.pos_ids = p.pos_ids;
  a.bufs = p.bufs;
  a.part_keys = p.part_keys;
  a.gtau = p.gtau;
  a.tau_in = p.tau_in;
  a.tau_stride = p.tau_stride;
  a.cand = p.cand;
  a.cand_cnt = p.cand_cnt;
  a.cand_cap = p.cand_cap;
  a.only_flagged = p.only_flagged;
  a.qmap = p.qmap;
  a.n_active = p.n_active;
  a.gmax = p.gmax;
  const int mode = p.gmax ? kGmax : (p.tau_in ? kFixed : kRunning);
  a.debug_no_topk = getenv("ASTRA_TC_DEBUG_NO_TOPK") != nullptr;
  static unsigned long long* dbg_buf = nullptr;
  const bool counters = getenv("ASTRA_TC_DEBUG_COUNTERS") != nullptr;
  if (counters && !dbg_buf) cudaMalloc(&dbg_buf, 12 * sizeof(unsigned long long));
  a.dbg = counters ? dbg_buf : nullptr;
  if (counters) cudaMemsetAsync(dbg_buf, 0, 12 * sizeof(unsigned long long), st);
  if (mode == kRunning) ASTRA_TRY(check_cuda(cudaMemsetAsync(p.gtau, 0, sizeof(uint64_t) * p.nq, st), "memset gtau"));
  const dim3 grid(static_cast<unsigned>(G));
  int rc;
  // CTA pairs (tcgen05 cta_group::2, M=256 per MMA, each CTA stages half of the
  // W tile) by default; ASTRA_TC_PAIR=0 selects W multicast in clusters of 2.
  // ncu: 1/3 less L2->SM traffic, tensor pipe 87% vs 85% active at the same
  // power-capped clock (profiles/r01/ncu_full_refresh_threshold_pair.txt).
  const bool pair = refresh_tc_pair();
  auto dispatch = [&](auto f8_tag) {
    constexpr bool F8 = decltype(f8_tag)::value;
    if (cl == 2 && pair) {
      if (mode == kFixed) return launch_variant<2, kFixed, true, F8>(tmA, tmB, a, grid, st);
      if (mode == kGmax) return launch_variant<2, kGmax, true, F8>(tmA, tmB, a, grid, st);
      return launch_variant<2, kRunning, true, F8>(tmA, tmB, a, grid, st);
    }
    if (mode == kFixed)
      return cl == 2 ? launch_variant<2, kFixed, false, F8>(tmA, tmB, a, grid, st)
                     : launch_variant<1, kFixed, false, F8>(tmA, tmB, a, grid, st);
    if (mode == kGmax)
      return cl == 2 ? launch_variant<2, kGmax, false, F8>(tmA, tmB, a, grid, st)
                     : launch_variant<1, kGmax, false, F8>(tmA, tmB, a, grid, st);
    return cl == 2 ? launch_variant<2, kRunning, false, F8>(tmA, tmB, a, grid, st)
                   : launch_variant<1, kRunning, false, F8>(tmA, tmB, a, grid, st);
  };
  rc = p.f8 ? dispatch(std::true_type()) : dispatch(std::false_type());
  if (counters && rc == ASTRA_OK) {
    unsigned long long h[12];
    cudaMemcpyAsync(h, dbg_buf, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const double ew = static_cast<double>(G) * kEpiWarps, mw = G;
    fprintf(stderr, "[refresh_tc %s] nq=%lld k=%d stride=%lld slow_steps=%llu/%llu (%.3f) compactions=%llu\n",
            mode == kFixed ? "fixed" : (mode == kGmax ? "gmax" : "running"), (long long)p.nq, p.k, (long long)p.tile_stride, h[0], h[3],
            h[3] ? double(h[0]) / h[3] : 0.0, h[2]);
    fprintf(stderr,
            "[refresh_tc] per epilogue warp Mcycles: total %.2f tfull-wait %.2f fast %.2f slow %.2f settle %.2f | "
            "per MMA warp: total %.2f tempty-wait %.2f full-wait %.2f\n",
            h[8] / ew / 1e6, h[4] / ew / 1e6, h[5] / ew / 1e6, h[6] / ew / 1e6, h[7] / ew / 1e6, h[11] / mw / 1e6,
            h[9] / mw / 1e6, h[10] / mw / 1e6);
  }
  return rc;
}

}  // namespace astra
