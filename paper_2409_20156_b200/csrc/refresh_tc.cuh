// refresh_tc.cuh — host interface of the tcgen05 refresh kernel (refresh_tc.cu),
// used by the orchestration in refresh.cu.
#pragma once

#include "common.cuh"

namespace astra {

// One launch of refresh_tc_kernel. Three epilogue modes:
//  * running (tau_in == nullptr): exact per-query running top-k of every
//    label tile swept (topk.cuh), one sorted list of k keys per (query, part)
//    in part_keys [n_parts][nq][k];
//  * fixed (tau_in != nullptr): every key >= the query's threshold
//    tau_in[q * tau_stride] is appended to cand [n_parts][nq][cand_cap], the
//    count (possibly > cand_cap: overflow) to cand_cnt [n_parts][nq];
//  * gmax (gmax != nullptr): the maximum score of every 64-label group of the
//    swept tiles, as orderable bits, to gmax [nq][n_swept_tiles * 4].
// tile_stride > 1 sweeps only every tile_stride-th 256-label tile (the sample
// pass). only_flagged (running mode): CTAs whose query tiles hold no flagged
// query exit at once (the verification fallback).
struct TcLaunch {
  const void* qb = nullptr;  // queries [nq, d]: bf16, or e4m3 bytes when f8
  int64_t nq = 0;
  int d = 0;
  const void* wb = nullptr;  // labels [L, d]: bf16, or e4m3 bytes when f8
  bool f8 = false;           // kind::f8f6f4 with e4m3 operands (d % 128 == 0)
  int64_t L = 0, off = 0;
  const int64_t* pos_indptr = nullptr;
  const int32_t* pos_ids = nullptr;
  int k = 0, cap = 0;
  uint64_t* bufs = nullptr;
  uint64_t* part_keys = nullptr;
  uint64_t* gtau = nullptr;
  int64_t tile_stride = 1;
  const uint64_t* tau_in = nullptr;
  int tau_stride = 1;
  uint64_t* cand = nullptr;
  int32_t* cand_cnt = nullptr;
  int cand_cap = 0;
  const int32_t* only_flagged = nullptr;
  uint32_t* gmax = nullptr;
  // compact verify (running mode): the first *n_active rows of qb are the
  // flagged queries, qmap[row] their original index (positives); the layout
  // uses n_parts_fixed label parts over every SM pair
  const int32_t* qmap = nullptr;
  const int32_t* n_active = nullptr;
  int n_parts_fixed = 0;
};

constexpr int kTcTileLabels = 256;

int launch_refresh_tc(const TcLaunch& p, cudaStream_t st);
// CTAs and per-query lists (= label parts) for nq queries over n_tiles label tiles.
void refresh_tc_layout(int64_t nq, int64_t n_tiles, int* n_ctas, int* n_parts);
// Cap on the SMs the refresh GEMM occupies (0 = all), so that a refresh on a
// side stream leaves SMs to the training step (astra_set_refresh_sm_budget).
void set_refresh_sm_budget(int n_sms);

}  // namespace astra
