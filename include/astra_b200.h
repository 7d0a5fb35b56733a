/*
 * astra_b200.h — C-ABI of the B200-native ASTRA classifier hot path.
 *
 * The reference (xcmix, pure Python/NumPy) has no FFI for this path: its
 * boundary is the Python call surface listed in SURVEY.md §8(b). Each entry
 * point below replaces the numeric core of one of those Python functions;
 * the Python mirror in paper_2409_20156_b200/ binds them with ctypes and
 * keeps the reference signatures, argument meanings and error classes.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers owned by the caller, row-major,
 *     unless stated otherwise. `stream` is a cudaStream_t passed as void*
 *     (NULL = legacy default stream). Calls are stream-ordered and never
 *     synchronise the host, except the *_sync helpers.
 *   - Status codes mirror xcmix.errors (errors.py:10-21), which the reference
 *     CLI maps to exit codes 2/3/4 (cli.py:91-105):
 *       0 ok, 2 ConfigError, 3 DataError, 4 NumericalError, 5 CUDA failure.
 *     astra_last_error() returns the message of the last failing call on the
 *     calling host thread.
 *   - Label ids are int32 (L < 2^31, which covers the 120M-label config).
 *   - "Key" = packed uint64 ordering used by every top-k in this library:
 *       key = (monotone_u32(score + 0.0f) << 32) | (0xFFFFFFFF - label_id)
 *     so the larger key is the higher score, ties toward the lower id — the
 *     reference's deterministic order (anns.py:103-109, anns.py:112-133).
 *     Key 0 marks an empty slot.
 */
#ifndef ASTRA_B200_H
#define ASTRA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASTRA_OK 0
#define ASTRA_ERR_CONFIG 2    /* xcmix.errors.ConfigError    */
#define ASTRA_ERR_DATA 3      /* xcmix.errors.DataError      */
#define ASTRA_ERR_NUMERICAL 4 /* xcmix.errors.NumericalError */
#define ASTRA_ERR_CUDA 5      /* CUDA runtime failure        */

/* Slot origin codes, loss.py:27-30; IMP is the importance-sampled extension. */
#define ASTRA_ORIGIN_POS 0
#define ASTRA_ORIGIN_HARD 1
#define ASTRA_ORIGIN_RAND 2
#define ASTRA_ORIGIN_PAD 3
#define ASTRA_ORIGIN_IMP 4

/* Refresh score modes. */
#define ASTRA_REFRESH_FP32_EXACT 0  /* SIMT fmaf, fixed k order: bit-exact ids    */
#define ASTRA_REFRESH_BF16 1        /* tcgen05 bf16 GEMM + top-k epilogue         */
#define ASTRA_REFRESH_BF16_RERANK 2 /* bf16 top-k' then fp32-exact re-rank to k   */
#define ASTRA_REFRESH_FP8_RERANK 3  /* e4m3 top-k' (2x tensor rate) then re-rank   */

/* Classifier storage / optimizer. */
#define ASTRA_W_FP32 0
#define ASTRA_W_BF16 1
#define ASTRA_OPT_SGD 0  /* classifiers.py:75-82: w <- w - lr*(g + wd*w)            */
#define ASTRA_OPT_ADAM 1 /* lazy sparse Adam (torch.optim.SparseAdam semantics)    */

/* Device status words written by astra_slate_step (int32[ASTRA_STATUS_WORDS]). */
#define ASTRA_STATUS_WORDS 4
#define ASTRA_STATUS_NONFINITE_GRAD 0     /* a touched row's gradient is non-finite */
#define ASTRA_STATUS_NONFINITE_GRAD_EMB 1 /* grad_emb is non-finite                  */
#define ASTRA_STATUS_BOUND_UNSAFE 2       /* overflow bound tripped -> checked path  */
#define ASTRA_STATUS_ID_RANGE 3           /* an id fell outside [0, n_labels_total)  */

const char* astra_version(void);
const char* astra_last_error(void);
/* Fills SM count and compute capability of the current device. */
int astra_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* Number of kernels this library launched on the calling process (all threads). */
uint64_t astra_launch_count(void);

/* Live kernel timing (bench.py's roofline). While enabled, the library records
 * a CUDA event pair on the launching stream around each launch of the named
 * kernels: "refresh_gemm" (the fused tcgen05 GEMM + selection pass that scores
 * every label: the threshold pass, or the single running-top-k pass),
 * "refresh_verify" (the two-pass plan's exact fallback pass), "step_single"
 * (the single label-major step pass), "slot_forward" and "label_update" (the
 * two-kernel step schedule), "gemm_f32" (astra_gemm_f32's tensor-core GEMM
 * kernel). Enabling fills a pool of events once (no event creation between
 * timed launches). astra_kernel_timing syncs the pairs recorded under `name`,
 * returns their summed milliseconds and count, clears them and returns the
 * events to the pool. Not a reference interface (measurement only).
 *
 * (Launch note: the step's kernels, astra_sample_slates -> astra_slate_step,
 * use programmatic dependent launch: each waits for its predecessor grid on
 * entry, so stream order is kept; ASTRA_PDL=0 launches them plainly.) */
void astra_kernel_timing_enable(int on);

/* Cap the number of SMs the refresh GEMM kernels occupy (0 = all SMs; the
 * default). The kernels are persistent (one CTA per SM of the budget), so a
 * refresh issued on a side stream leaves the other SMs to the training step
 * running concurrently on the main stream — the B200 form of the reference's
 * background refresh thread (trainer.py:198-214). Process-wide setting. */
void astra_set_refresh_sm_budget(int n_sms);

/* Step schedule (process-wide). on = 0 (default): for d % 128 == 0 (d <= 768)
 * with a w_absmax bound, astra_slate_step runs ONE label-major pass that reads
 * and writes each touched W row once and adds each slot's f * W_row into
 * grad_emb with fp32 vector reductions: W', the loss and the factors are
 * deterministic (W' bit-identical to the two-kernel schedule), grad_emb's
 * summation order is not; labels with more than 32 occurrences in the batch
 * are updated by a CTA each beside the pass (same order and roundings).
 * SGD and Adam alike (ASTRA_STEP_SINGLE_ADAM=0 keeps Adam on the two-kernel
 * schedule). on = 1: the two-kernel schedule (slot-major gather
 * forward, then the label-major update), bitwise run-to-run deterministic.
 * The environment variable ASTRA_STEP_SINGLE=0 is equivalent to on = 1. */
void astra_set_step_deterministic(int on);
int astra_kernel_timing(const char* name, double* total_ms, int64_t* count);

/* fp32 -> bf16 (round-to-nearest-even), n elements. Used for W/query snapshots. */
int astra_f32_to_bf16(const float* src, uint16_t* dst, int64_t n, void* stream);

/* ------------------------------------------------------------------------
 * Shortlist refresh — replaces the exact branch of
 *   retrieve_hard_negatives(index, embeddings, positives, k_h)   anns.py:233-256
 * including the positive mask (anns.py:254-255) and _batched_topk
 * (anns.py:112-133). Per query: the k largest scores over the label shard
 * [label_offset, label_offset + n_labels) excluding the query's positives,
 * descending, ties toward the lower id. Scores never reach HBM.
 *
 *   queries_f32   nq x d   fp32 (FP32_EXACT, BF16_RERANK; may be NULL for BF16
 *                          if queries_bf16 is given)
 *   queries_bf16  nq x d   bf16 bits, or NULL (converted into the workspace)
 *   labels_f32    n_labels x d fp32 snapshot (FP32_EXACT, BF16_RERANK; for
 *                 BF16_RERANK it may be NULL: the re-rank then scores the bf16
 *                 snapshot's values exactly — the bf16-W configuration)
 *   labels_bf16   n_labels x d bf16 snapshot (BF16, BF16_RERANK; the re-rank
 *                 rows of FP8_RERANK when labels_f32 is NULL)
 *   labels_e4m3   n_labels x d e4m3 snapshot (FP8_RERANK: astra_quantize_e4m3),
 *                 or NULL
 *   pos_indptr    nq+1 int64, pos_ids int32 GLOBAL ids sorted ascending per row
 *   out_keys      nq x k packed keys (input of astra_topk_merge), or NULL
 *   out_ids       nq x k int32 global ids, or NULL
 *   out_scores    nq x k fp32 scores (fp32-exact in modes 0/2/3), or NULL
 * A query with fewer than k admissible labels in the shard is padded with
 * key 0 / id -1 / score -inf (the cross-shard merge then fills it).
 * Constraints: 1 <= k <= 2048; BF16 modes need d % 64 == 0; FP8_RERANK needs
 * d % 128 == 0, k <= 240 (k' = max(2k, k+32) <= 512) and fp32 queries.
 * ------------------------------------------------------------------------ */
size_t astra_refresh_workspace_size(int64_t nq, int64_t n_labels, int d, int k, int mode);
int astra_refresh_topk(const float* queries_f32, const uint16_t* queries_bf16, int64_t nq, int d,
                       const float* labels_f32, const uint16_t* labels_bf16, const uint8_t* labels_e4m3,
                       int64_t n_labels, int64_t label_offset, const int64_t* pos_indptr,
                       const int32_t* pos_ids, int k, int mode, uint64_t* out_keys, int32_t* out_ids,
                       float* out_scores, void* workspace, size_t workspace_bytes, void* stream);

/* The e4m3 label snapshot for ASTRA_REFRESH_FP8_RERANK (build_exact's copy,
 * anns.py:99-100, in the tensor cores' 8-bit format): n values of src (fp32,
 * or bf16 when src_bf16; n % 4 == 0, 16-byte aligned) -> dst bytes
 * e4m3(x * 448 / max|x|), round-to-nearest-even, saturating. max|x| is
 * reduced on the device (no host sync); scratch = 2 device floats, scratch[1]
 * receives the scale. One scale for all labels multiplies every score alike,
 * so rankings are those of the unscaled e4m3 values. */
int astra_quantize_e4m3(const void* src, int src_bf16, int64_t n, uint8_t* dst, float* scratch, void* stream);

/* Diagnostic of the last astra_refresh_topk call made with `workspace` and
 * the same (nq, n_labels, d, k, mode): how many queries the two-pass plan
 * could not prove exact from its threshold candidates (they were recomputed
 * by the exact running top-k, so the result is exact either way). *out_count
 * = -1 when that shape does not use the two-pass plan. Synchronises `stream`.
 * No reference counterpart (observability of anns.py:233-256's replacement). */
int astra_refresh_flagged(const void* workspace, size_t workspace_bytes, int64_t nq, int64_t n_labels, int d,
                          int k, int mode, int64_t* out_count, void* stream);

/* Merge n_parts partial top-k lists per query (layout [n_parts][nq][k_in],
 * e.g. an all-gather over label shards) into the global top-k_out. Each list
 * must be sorted descending and zero-padded, as astra_refresh_topk writes its
 * out_keys. Exact: the result equals a single-shard refresh over the union of
 * the shards. */
size_t astra_merge_workspace_size(int64_t nq, int k_out);
int astra_topk_merge(const uint64_t* part_keys, int64_t nq, int n_parts, int k_in, int k_out,
                     uint64_t* out_keys, int32_t* out_ids, float* out_scores, void* workspace,
                     size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Negative-mixture sampler — replaces _assemble_batch_slates
 * (trainer.py:262-318) / assemble_slate (sampler.py:146-186) with a
 * counter-based Philox4x32-10 stream keyed by (seed, epoch, step, row, slot).
 * Slot layout per row (S = k_p + k_h + k_i + k_r):
 *   [0, k_p)            positives: uniform k_p-subset in random order; rows with
 *                       fewer positives are padded by uniform non-positive labels
 *                       (trainer.py:273-290). origin POS / PAD, y = 1 / 0.
 *   [k_p, +k_h)         hard: hard[b, 0:k_h] verbatim (trainer.py:295-298), y = 0.
 *   [.., +k_i)          importance (extension): draws from cand[b, 0:n_c] with
 *                       probabilities cand_q; weight 1/(k_i q); origin IMP.
 *   [.., +k_r)          uniform with replacement over [L] \ C, C = hard (+cand),
 *                       rank->id map over sorted C (trainer.py:300-306),
 *                       weight (L-|C|)/k_r (trainer.py:315-317),
 *                       y = id in positives (trainer.py:309).
 * Outputs are B x S (ids int32, y int8, origin int8, weights fp32).
 * hard rows must hold distinct ids; cand rows distinct and disjoint from hard.
 * ------------------------------------------------------------------------ */
int astra_sample_slates(uint64_t seed, uint32_t epoch, uint32_t step, const int64_t* rows, int B,
                        const int64_t* pos_indptr, const int32_t* pos_ids, const int32_t* hard,
                        int hard_stride, int k_h, const int32_t* cand, const float* cand_q,
                        int cand_stride, int n_c, int k_i, int64_t n_labels, int k_p, int k_r,
                        int32_t* ids, int8_t* y, int8_t* origin, float* weights, void* stream);

/* Importance-sampled class (extension): split a stale
 * refresh of top-(k_h + n_c) per row (ids int32 + fp32 scores [nq, k_tot],
 * descending, as astra_refresh_topk writes them, k_tot = k_h + n_c) into the
 * sampler's inputs: hard [nq, k_h] (H, the first k_h ids), cand [nq, n_c]
 * (C, the next n_c) and cand_q [nq, n_c] = sigmoid(stale score) (unnormalised
 * draw weights; astra_sample_slates normalises per row and weights each draw
 * 1/(k_i q)). ids < 0 get q = 0. H and C are disjoint and exclude the row's
 * positives (the refresh masked them). */
int astra_importance_split(const int32_t* ids, const float* scores, int64_t nq, int k_tot, int k_h,
                           int32_t* hard, int32_t* cand, float* cand_q, void* stream);

/* ------------------------------------------------------------------------
 * Sampled BCE forward/backward fused with the sparse row update — replaces
 * the classifier half of _batch_forward_backward (trainer.py:366-394) and
 * apply_classifier_updates_arrays (classifiers.py:75-82).
 *   emb        B x d fp32  embeddings AFTER dropout (emb_used, trainer.py:343-348)
 *   keep       B x d fp32  dropout keep scale or NULL (grad_emb *= keep, :383-384)
 *   ids/y      B x S       slates (global ids)
 *   origin     origin_row_stride = 0: one S-vector shared by every row (the
 *              reference's row-0 origin, trainer.py:313); = S: per-row origin
 *   weights    weights_row_stride = 0 (S-vector) or S (per-row)
 *   factors_in B x S fp32 or NULL: if given, skip the score/factor stage and
 *              use these d(loss)/d(score) factors (parity tests feed the
 *              reference's factors to check the update bit-for-bit)
 *   W          n_labels_local x d (fp32 or bf16); slots whose id falls outside
 *              [label_offset, label_offset + n_labels_local) belong to another
 *              shard and are skipped (label-range sharding)
 *   adam_m/v   n_labels_local x d fp32 (ASTRA_OPT_ADAM) or NULL
 *   grad_emb   B x d fp32 out (partial over this shard's slots)
 *   loss_out   1 fp64 out: sum of this shard's slate loss terms (fp64)
 *   status     int32[ASTRA_STATUS_WORDS] out (zeroed by the call)
 *   factors_out B x S fp32 out (d(loss)/d(score) per slot) or NULL
 *   w_absmax   1 fp32 in/out or NULL: a running upper bound on max|W| of this
 *              shard, kept current by the call (every updated row folds its
 *              new |values| in). With it (SGD, d % 128 == 0, d <= 768, 16-byte
 *              aligned emb/W/grad_emb, astra_set_step_deterministic(0)), the
 *              call proves on the device that no gradient and no grad_emb
 *              entry can overflow and runs the single label-major pass
 *              (each touched row read and written once; grad_emb reduced in
 *              arrival order); without it, or when the proof fails, it runs
 *              the deterministic two-kernel schedule (slot-major gather
 *              forward, then the label-major update), which is also the Adam
 *              schedule. The schedule kernels not taken return at once.
 *   lr, weight_decay, betas, eps are host doubles: SGD rounds lr/wd to fp32
 *   like np.float32(lr) (classifiers.py:82); Adam derives its step size in
 *   double like torch.optim.SparseAdam.
 * Semantics: every id present in the slate is updated once (dead/pad slots
 * included, so they receive weight decay), gradients sum duplicates in
 * ascending flat (b*S+s) order, W is updated only if every touched row's
 * gradient and grad_emb are finite (the reference raises before writing).
 * ------------------------------------------------------------------------ */
size_t astra_step_workspace_size(int B, int S, int d, int64_t n_labels_local);
int astra_slate_step(const float* emb, const float* keep, const int32_t* ids, const int8_t* y,
                     const int8_t* origin, int64_t origin_row_stride, const float* weights,
                     int64_t weights_row_stride, const float* factors_in, int B, int S, int d,
                     void* W, int w_dtype, float* adam_m, float* adam_v, int optimizer,
                     int64_t n_labels_local, int64_t label_offset, double lr, double weight_decay,
                     double adam_beta1, double adam_beta2, double adam_eps, int64_t adam_step,
                     float* grad_emb, double* loss_out, int32_t* status, float* factors_out,
                     float* w_absmax, void* workspace, size_t workspace_bytes, void* stream);

/* apply_classifier_updates_arrays(bank, ids, grads, lr, wd)  classifiers.py:75-82
 * ids (U, unique, local row index) and grads (U x d) on device. Raises
 * NumericalError semantics: nothing is written if any gradient is
 * non-finite (status[0] = 1, return 0 — the caller syncs and raises). */
int astra_apply_updates(void* W, int w_dtype, int64_t n_labels, int d, const int64_t* ids,
                        const float* grads, int64_t U, float lr, float weight_decay,
                        int32_t* status, void* stream);

/* ------------------------------------------------------------------------
 * All-negatives (full-loss) arm, train_full_loss_baseline (trainer.py:563-616),
 * and the dense probe loss, _probe_full_loss (trainer.py:398-403). The arm's
 * fp32 GEMMs (E W^T, G W, G^T E: trainer.py:593-606) run on the tf32 tensor
 * cores split three ways (astra_gemm_f32); the elementwise parts follow.
 *
 * astra_dense_bce: scores B x n_labels (fp32, or fp64 when scores_f64), the
 * positives as a CSR (pos_indptr[B+1] int64, pos_ids int32, sorted distinct
 * per row). Writes G = f32(0.5 (1 + tanh(s / 2))) - y (trainer.py:597; G may
 * be NULL: loss only) and *loss_out = float64 sum of y sp(-s) + (1-y) sp(s)
 * (trainer.py:595 / :401-402). Deterministic (fixed-order reductions).
 * Workspace: astra_dense_workspace_size(B) bytes. */
size_t astra_dense_workspace_size(int B);
int astra_dense_bce(const void* scores, int scores_f64, int B, int64_t n_labels,
                    const int64_t* pos_indptr, const int32_t* pos_ids, float* G,
                    double* loss_out, void* workspace, size_t workspace_bytes, void* stream);

/* Dense SGD over n elements: W -= f32(lr) * (grads + f32(wd) * W), each op
 * rounded like NumPy (trainer.py:604-606; no finiteness check, as there). */
int astra_dense_sgd(float* W, const float* grads, int64_t n, float lr, float weight_decay,
                    void* stream);

/* The label-sharded BF16 candidate pass with a global threshold (the
 * multi-GPU refresh, engine._refresh_sharded): each shard's sample statistics
 * go to the rows' owners, which return a global per-query threshold; the
 * shard's candidates at or above it are selected locally and the owners'
 * summed counts decide which queries take the exact verify pass. The
 * workspace is astra_refresh_workspace_size(nq, n_labels, d, k,
 * ASTRA_REFRESH_BF16); k is the candidate count (k').
 *   astra_refresh_plan_j: j of the sample statistics for this shape (0 = the
 *     shape does not run the two-pass plan: use astra_refresh_topk).
 *   stage 1: sample_top [nq, j] = the shard's j largest sampled 64-label
 *     group maxima per query (orderable score bits, any order).
 *   stage 2: tau_keys [nq] (the global threshold, key form score << 32) ->
 *     io_keys [nq, k] = the shard's best non-positive candidates at or above
 *     it (descending, 0-padded), counts [nq] = how many (<= k), flags [nq] =
 *     1 where a candidate list overflowed (verify needed whatever the counts).
 *   stage 3: flags [nq] (the global verify set) -> io_keys rows of the
 *     flagged queries replaced by the shard's exact top-k. */
int astra_refresh_plan_j(int64_t nq, int64_t n_labels, int d, int k);
int astra_refresh_sharded_stage(int stage, const float* queries_f32, const uint16_t* queries_bf16, int64_t nq, int d,
                                const uint16_t* labels_bf16, int64_t n_labels, int64_t label_offset,
                                const int64_t* pos_indptr, const int32_t* pos_ids, int k, uint32_t* sample_top,
                                const uint64_t* tau_keys, uint64_t* io_keys, int32_t* counts, int32_t* flags,
                                void* workspace, size_t workspace_bytes, void* stream);

/* The refresh's fp32 re-rank on its own (the last stage of BF16_RERANK,
 * anns.py:253-256 scores): for each of nq queries (fp32 [nq, d]) score the
 * kc candidate keys cand[q * kc + j] (astra key format; 0 = no candidate)
 * against the label rows (fp32, or bf16 when w_dtype = ASTRA_W_BF16; [L_local,
 * d], candidate id - label_offset = row) with the FP32_EXACT fmaf order and
 * write the best k (k <= kc) as keys / ids / scores (-1 / -inf past the
 * candidates). Used by the label-sharded refresh: each shard re-ranks only its
 * candidates at or above the global k'-th bf16 key. */
int astra_rerank_candidates(const float* queries, int64_t nq, int d, const uint64_t* cand, int kc,
                            const void* labels, int w_dtype, int64_t label_offset, int k, uint64_t* out_keys,
                            int32_t* out_ids, float* out_scores, void* stream);

/* D[M, N] = A B^T in fp32 accuracy on the tf32 tensor cores (3xTF32: each
 * operand split into a tf32 hi part and an fp32 remainder; hi*hi + lo*hi +
 * hi*lo accumulated in fp32; replaces the host's numpy sgemm of the
 * full-loss arm, trainer.py:593-606). A is [M, K] row-major (a_kmajor = 1)
 * or given transposed as [K, M] row-major (a_kmajor = 0); B likewise [N, K]
 * or [K, N]. D is [M, N] row-major, overwritten. Summation order differs from
 * a sequential sgemm: results agree to fp32 rounding of the sum (tolerance
 * 1e-5 relative in the tests). Workspace: astra_gemm_f32_workspace_size. */
size_t astra_gemm_f32_workspace_size(int64_t M, int64_t N, int64_t K);
int astra_gemm_f32(const float* A, int a_kmajor, const float* B, int b_kmajor, int64_t M, int64_t N, int64_t K,
                   float* D, void* workspace, size_t workspace_bytes, void* stream);

/* Synchronous helper: cudaStreamSynchronize + error mapping. */
int astra_stream_sync(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ASTRA_B200_H */
