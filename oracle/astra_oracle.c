/*
 * astra_oracle.c — CPU restatement used as the CHECKER for the CUDA path.
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library. The product never links it.
 *
 * Two pieces whose bits the GPU must reproduce exactly:
 *
 * 1. oracle_refresh_fp32 — the exact shortlist refresh of
 *    retrieve_hard_negatives (anns.py:233-256): per query, drop the query's
 *    positives (anns.py:254-255) and keep the top-k labels by score,
 *    descending, ties to the lower id (anns.py:103-109, :112-133).
 *    The reference scores with OpenBLAS sgemm (anns.py:253), whose summation
 *    order is not reproducible; this restatement fixes the order instead:
 *        s = 0; for t in 0..d-1: s = fmaf(q[t], w[t], s)
 *    (correctly rounded on both CPU and GPU), so shortlist ids can be
 *    compared bit-for-bit. Against the reference's own sgemm ids the tests
 *    compare up to score ties.
 *
 * 2. oracle_sample_slates — the Philox4x32-10 negative-mixture sampler that
 *    replaces the reference's PCG64 stream in _assemble_batch_slates
 *    (trainer.py:262-318). The reference's stream cannot be reproduced, so
 *    the distributional contract is validated statistically (the reference's
 *    own sampler tests, test_sampler.py:104-136) and the GPU kernel must match
 *    this restatement draw-for-draw. The counter layout is the spec:
 *      key     = (seed_lo32, seed_hi32)
 *      counter = (c0, row_lo32, epoch, (tag << 24) | (step & 0xFFFFFF))
 *      TAG_POSKEY=1  c0 = positive index         -> u32 sort key (random subset)
 *      TAG_PAD   =2  c0 = slot | attempt << 20   -> label in [0, L), reject positives
 *      TAG_IMP   =3  c0 = slot                   -> inverse-CDF over stored q
 *      TAG_RAND  =4  c0 = slot                   -> v in [0, L-|C|), rank->id map
 *    Bounded draws use the 128-bit product of a 64-bit uniform (out.x | out.y<<32)
 *    with the range (no modulo bias beyond range/2^64).
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off, no fast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ keys */

static inline uint32_t ord_f32(float s) {
  s = s + 0.0f; /* -0.0 -> +0.0 */
  uint32_t b;
  memcpy(&b, &s, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

static inline uint64_t make_key(float s, int64_t id) {
  return ((uint64_t)ord_f32(s) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)id);
}

static inline float key_score(uint64_t key) {
  uint32_t o = (uint32_t)(key >> 32);
  uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  float s;
  memcpy(&s, &b, 4);
  return s;
}

static inline int32_t key_id(uint64_t key) { return (int32_t)(0xFFFFFFFFu - (uint32_t)key); }

static int cmp_key_desc(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x < y) - (x > y);
}

static int is_member(const int32_t* sorted, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < n && sorted[lo] == v;
}

/* ------------------------------------------------------------ refresh */

void oracle_refresh_fp32(const float* Q, int64_t nq, int d, const float* W, int64_t L,
                         int64_t label_offset, const int64_t* pos_indptr, const int32_t* pos_ids, int k,
                         uint64_t* out_keys, int32_t* out_ids, float* out_scores) {
#pragma omp parallel
  {
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(L > 0 ? L : 1));
#pragma omp for schedule(dynamic, 4)
    for (int64_t i = 0; i < nq; ++i) {
      const float* q = Q + (size_t)i * d;
      const int32_t* pos = pos_ids + pos_indptr[i];
      int64_t npos = pos_indptr[i + 1] - pos_indptr[i];
      int64_t m = 0;
      for (int64_t l = 0; l < L; ++l) {
        int64_t gid = l + label_offset;
        if (is_member(pos, npos, gid)) continue;
        const float* w = W + (size_t)l * d;
        float s = 0.0f;
        for (int t = 0; t < d; ++t) s = fmaf(q[t], w[t], s);
        keys[m++] = make_key(s, gid);
      }
      qsort(keys, (size_t)m, sizeof(uint64_t), cmp_key_desc);
      for (int j = 0; j < k; ++j) {
        uint64_t key = j < m ? keys[j] : 0;
        if (out_keys) out_keys[i * k + j] = key;
        if (out_ids) out_ids[i * k + j] = key ? key_id(key) : -1;
        if (out_scores) out_scores[i * k + j] = key ? key_score(key) : -INFINITY;
      }
    }
    free(keys);
  }
}

/* fp32 scores with the same fixed order, for recall / tolerance checks. */
void oracle_scores_fp32(const float* Q, int64_t nq, int d, const float* W, int64_t L, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nq; ++i)
    for (int64_t l = 0; l < L; ++l) {
      float s = 0.0f;
      for (int t = 0; t < d; ++t) s = fmaf(Q[(size_t)i * d + t], W[(size_t)l * d + t], s);
      out[(size_t)i * L + l] = s;
    }
}

/* ------------------------------------------------------------ Philox */

typedef struct {
  uint32_t v[4];
} u32x4;

static inline u32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                  uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  u32x4 o = {{c0, c1, c2, c3}};
  return o;
}

enum { TAG_POSKEY = 1, TAG_PAD = 2, TAG_IMP = 3, TAG_RAND = 4 };

typedef struct {
  uint32_t k0, k1, row, epoch, step;
} philox_ctx;

static inline u32x4 draw(const philox_ctx* c, uint32_t c0, uint32_t tag) {
  return philox4x32_10(c0, c->row, c->epoch, (tag << 24) | (c->step & 0xFFFFFFu), c->k0, c->k1);
}

static inline uint64_t bounded(u32x4 r, uint64_t n) {
  uint64_t x = (uint64_t)r.v[0] | ((uint64_t)r.v[1] << 32);
  return (uint64_t)(((unsigned __int128)x * n) >> 64);
}

/* exported for the bit-exact Philox known-answer test */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  u32x4 r = philox4x32_10(ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1]);
  memcpy(out, r.v, 16);
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

typedef struct {
  uint32_t key;
  int32_t idx;
} keyidx;

static int cmp_keyidx(const void* a, const void* b) {
  const keyidx* x = (const keyidx*)a;
  const keyidx* y = (const keyidx*)b;
  if (x->key != y->key) return (x->key > y->key) - (x->key < y->key);
  return (x->idx > y->idx) - (x->idx < y->idx);
}

/* Mirrors astra_sample_slates (include/astra_b200.h); see the header comment
 * for the counter layout. Returns 0, or 2 (ConfigError) on an infeasible
 * configuration. */
int oracle_sample_slates(uint64_t seed, uint32_t epoch, uint32_t step, const int64_t* rows, int B,
                         const int64_t* pos_indptr, const int32_t* pos_ids, const int32_t* hard,
                         int hard_stride, int k_h, const int32_t* cand, const float* cand_q,
                         int cand_stride, int n_c, int k_i, int64_t L, int k_p, int k_r, int32_t* ids,
                         int8_t* y, int8_t* origin, float* weights) {
  const int S = k_p + k_h + k_i + k_r;
  const int use_cand = k_i > 0 && n_c > 0;
  const int m = k_h + (use_cand ? n_c : 0);
  if (m >= L) return 2;
  int32_t* C = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  int64_t* shifted = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  double* cdf = (double*)malloc(sizeof(double) * (size_t)(n_c > 0 ? n_c : 1));
  int64_t maxp = 1;
  for (int b = 0; b < B; ++b) {
    int64_t np = pos_indptr[b + 1] - pos_indptr[b];
    if (np > maxp) maxp = np;
  }
  keyidx* ki = (keyidx*)malloc(sizeof(keyidx) * (size_t)maxp);
  for (int b = 0; b < B; ++b) {
    philox_ctx cx = {(uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)rows[b], epoch, step};
    const int32_t* pos = pos_ids + pos_indptr[b];
    const int64_t npos = pos_indptr[b + 1] - pos_indptr[b];
    int32_t* oid = ids + (size_t)b * S;
    int8_t* oy = y + (size_t)b * S;
    int8_t* oo = origin + (size_t)b * S;
    float* ow = weights + (size_t)b * S;
    /* positives: random order by (philox key, index); first k_p (trainer.py:273-281) */
    for (int64_t p = 0; p < npos; ++p) {
      ki[p].key = draw(&cx, (uint32_t)p, TAG_POSKEY).v[0];
      ki[p].idx = (int32_t)p;
    }
    qsort(ki, (size_t)npos, sizeof(keyidx), cmp_keyidx);
    for (int j = 0; j < k_p; ++j) {
      if (j < npos) {
        oid[j] = pos[ki[j].idx];
        oy[j] = 1;
        oo[j] = 0; /* POS */
      } else {
        /* pad: uniform over [0, L) rejecting the row's positives (trainer.py:283-290) */
        uint32_t a = 0;
        int64_t v;
        do {
          v = (int64_t)bounded(draw(&cx, (uint32_t)j | (a << 20), TAG_PAD), (uint64_t)L);
          ++a;
        } while (is_member(pos, npos, v));
        oid[j] = (int32_t)v;
        oy[j] = 0;
        oo[j] = 3; /* PAD */
      }
      ow[j] = 1.0f;
    }
    /* hard (trainer.py:295-298) */
    for (int j = 0; j < k_h; ++j) {
      oid[k_p + j] = hard[(size_t)b * hard_stride + j];
      oy[k_p + j] = 0;
      oo[k_p + j] = 1; /* HARD */
      ow[k_p + j] = 1.0f;
    }
    /* importance extension */
    double tot = 0.0;
    if (use_cand) {
      for (int c = 0; c < n_c; ++c) {
        tot += (double)cand_q[(size_t)b * cand_stride + c];
        cdf[c] = tot;
      }
    }
    for (int j = 0; j < k_i; ++j) {
      int s = k_p + k_h + j;
      int c = 0;
      if (use_cand) {
        u32x4 r = draw(&cx, (uint32_t)s, TAG_IMP);
        uint64_t x = (uint64_t)r.v[0] | ((uint64_t)r.v[1] << 32);
        double u = (double)(x >> 11) * 0x1.0p-53;
        double target = u * tot;
        int lo = 0, hi = n_c - 1;
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (cdf[mid] > target)
            hi = mid;
          else
            lo = mid + 1;
        }
        c = lo;
      }
      int32_t id = use_cand ? cand[(size_t)b * cand_stride + c] : 0;
      double q = use_cand ? (double)cand_q[(size_t)b * cand_stride + c] : 1.0;
      oid[s] = id;
      oy[s] = (int8_t)is_member(pos, npos, id);
      oo[s] = 4; /* IMP */
      ow[s] = use_cand ? (float)(tot / ((double)k_i * q)) : 0.0f;
    }
    /* uniform over [L] \ C via the rank -> id map (trainer.py:300-306) */
    for (int j = 0; j < k_h; ++j) C[j] = hard[(size_t)b * hard_stride + j];
    if (use_cand)
      for (int c = 0; c < n_c; ++c) C[k_h + c] = cand[(size_t)b * cand_stride + c];
    qsort(C, (size_t)m, sizeof(int32_t), cmp_i32);
    for (int j = 0; j < m; ++j) shifted[j] = (int64_t)C[j] - j;
    float wr = k_r > 0 ? (float)((double)(L - m) / (double)k_r) : 0.0f;
    for (int j = 0; j < k_r; ++j) {
      int s = k_p + k_h + k_i + j;
      int64_t v = (int64_t)bounded(draw(&cx, (uint32_t)s, TAG_RAND), (uint64_t)(L - m));
      int lo = 0, hi = m; /* count of shifted <= v */
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (shifted[mid] <= v)
          lo = mid + 1;
        else
          hi = mid;
      }
      int64_t id = v + lo;
      oid[s] = (int32_t)id;
      oy[s] = (int8_t)is_member(pos, npos, id); /* trainer.py:309 */
      oo[s] = 2;                               /* RAND */
      ow[s] = wr;                              /* trainer.py:315-317 */
    }
  }
  free(C);
  free(shifted);
  free(cdf);
  free(ki);
  return 0;
}

/* ------------------------------------------------------------ refresh, blocked
 * oracle_refresh_fp32_blocked: the same result as oracle_refresh_fp32 (every
 * score is the same sequential fmaf chain over t = 0..d-1, so the keys are
 * bit-identical), organised for the production-size parity tests (L = 1.3M,
 * 15M): 16 queries x 4 labels of independent fmaf chains per step (the
 * compiler turns them into vector FMAs, each lane still a correctly rounded
 * fmaf; AVX2 FMA intrinsics), pthreads over (query block, label chunk) tasks, a size-k min-heap of
 * keys per query and task, then a merge. W may be fp32 or bf16 (uint16 bit
 * patterns, widened exactly). nthreads <= 0: one thread per online CPU. */
#include <immintrin.h>
#include <pthread.h>
#include <unistd.h>

#define QB 16
#define LB 4

static void heap_sift_down(uint64_t* h, int n, int i) {
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && h[l] < h[m]) m = l;
    if (r < n && h[r] < h[m]) m = r;
    if (m == i) return;
    uint64_t t = h[i];
    h[i] = h[m];
    h[m] = t;
    i = m;
  }
}

/* min-heap of at most k keys (smallest at h[0]); *n = current size */
static inline void heap_push(uint64_t* h, int* n, int k, uint64_t key) {
  if (*n < k) {
    int i = (*n)++;
    h[i] = key;
    while (i > 0) {
      int p = (i - 1) / 2;
      if (h[p] <= h[i]) break;
      uint64_t t = h[p];
      h[p] = h[i];
      h[i] = t;
      i = p;
    }
  } else if (key > h[0]) {
    h[0] = key;
    heap_sift_down(h, k, 0);
  }
}

static inline float bf16_bits_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

typedef struct {
  const float* Q;
  int64_t nq;
  int d;
  const void* W;
  int w_bf16;
  int64_t L, label_offset;
  const int64_t* pos_indptr;
  const int32_t* pos_ids;
  int k;
  int64_t nlc, lchunk, ntasks;
  uint64_t* heaps;
  int* hn;
  int64_t next; /* task counter (atomic) */
} blocked_ctx;

static void blocked_task(blocked_ctx* c, int64_t task, float* qt, float* wb) {
  const int d = c->d, k = c->k;
  int64_t qb = task / c->nlc, lc = task % c->nlc;
  int64_t q0 = qb * QB;
  int nqq = (int)(c->nq - q0 < QB ? c->nq - q0 : QB);
  for (int t = 0; t < d; ++t)
    for (int j = 0; j < QB; ++j) qt[(size_t)t * QB + j] = j < nqq ? c->Q[(size_t)(q0 + j) * d + t] : 0.0f;
  uint64_t* h = c->heaps + (size_t)task * QB * k;
  int* n = c->hn + task * QB;
  int64_t l0 = lc * c->lchunk, l1 = l0 + c->lchunk < c->L ? l0 + c->lchunk : c->L;
  for (int64_t l = l0; l < l1; l += LB) {
    int nl = (int)(l1 - l < LB ? l1 - l : LB);
    for (int i = 0; i < LB; ++i) {
      int64_t row = l + (i < nl ? i : 0);
      if (c->w_bf16) {
        const uint16_t* src = (const uint16_t*)c->W + (size_t)row * d;
        for (int t = 0; t < d; ++t) wb[(size_t)t * LB + i] = bf16_bits_to_f32(src[t]);
      } else {
        const float* src = (const float*)c->W + (size_t)row * d;
        for (int t = 0; t < d; ++t) wb[(size_t)t * LB + i] = src[t];
      }
    }
    /* s[i][j] = fmaf(q_j[t], w_i[t], s[i][j]) for t = 0..d-1: 8 independent
       vector FMA chains (each lane one correctly rounded fmaf) */
    __m256 acc[LB][2];
    for (int i = 0; i < LB; ++i) acc[i][0] = acc[i][1] = _mm256_setzero_ps();
    for (int t = 0; t < d; ++t) {
      __m256 q0v = _mm256_loadu_ps(qt + (size_t)t * QB), q1v = _mm256_loadu_ps(qt + (size_t)t * QB + 8);
      for (int i = 0; i < LB; ++i) {
        __m256 w = _mm256_broadcast_ss(wb + (size_t)t * LB + i);
        acc[i][0] = _mm256_fmadd_ps(q0v, w, acc[i][0]);
        acc[i][1] = _mm256_fmadd_ps(q1v, w, acc[i][1]);
      }
    }
    float s[LB][QB];
    for (int i = 0; i < LB; ++i) {
      _mm256_storeu_ps(s[i], acc[i][0]);
      _mm256_storeu_ps(s[i] + 8, acc[i][1]);
    }
    for (int i = 0; i < nl; ++i) {
      int64_t gid = l + i + c->label_offset;
      for (int j = 0; j < nqq; ++j) {
        int64_t qi = q0 + j;
        const int32_t* pos = c->pos_ids + c->pos_indptr[qi];
        if (is_member(pos, c->pos_indptr[qi + 1] - c->pos_indptr[qi], gid)) continue;
        heap_push(h + (size_t)j * k, &n[j], k, make_key(s[i][j], gid));
      }
    }
  }
}

static void* blocked_worker(void* arg) {
  blocked_ctx* c = (blocked_ctx*)arg;
  float* qt = (float*)malloc(sizeof(float) * (size_t)c->d * QB);
  float* wb = (float*)malloc(sizeof(float) * (size_t)c->d * LB);
  for (;;) {
    int64_t task = __atomic_fetch_add(&c->next, 1, __ATOMIC_RELAXED);
    if (task >= c->ntasks) break;
    blocked_task(c, task, qt, wb);
  }
  free(qt);
  free(wb);
  return NULL;
}

void oracle_refresh_fp32_blocked(const float* Q, int64_t nq, int d, const void* W, int w_bf16, int64_t L,
                                 int64_t label_offset, const int64_t* pos_indptr, const int32_t* pos_ids, int k,
                                 int nthreads, uint64_t* out_keys, int32_t* out_ids, float* out_scores) {
  if (k <= 0 || nq <= 0) return;
  int nth = nthreads > 0 ? nthreads : (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nth < 1) nth = 1;
  blocked_ctx c;
  memset(&c, 0, sizeof(c));
  c.Q = Q; c.nq = nq; c.d = d; c.W = W; c.w_bf16 = w_bf16; c.L = L; c.label_offset = label_offset;
  c.pos_indptr = pos_indptr; c.pos_ids = pos_ids; c.k = k;
  int64_t nqb = (nq + QB - 1) / QB;
  /* enough tasks for the threads: split the labels into chunks */
  c.nlc = (8 * (int64_t)nth + nqb - 1) / nqb;
  if (c.nlc > L / 1024 + 1) c.nlc = L / 1024 + 1;
  if (c.nlc < 1) c.nlc = 1;
  c.lchunk = (L + c.nlc - 1) / c.nlc;
  c.ntasks = nqb * c.nlc;
  c.heaps = (uint64_t*)calloc((size_t)(c.ntasks * QB * k), sizeof(uint64_t));
  c.hn = (int*)calloc((size_t)(c.ntasks * QB), sizeof(int));
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nth);
  for (int i = 0; i < nth; ++i) pthread_create(&th[i], NULL, blocked_worker, &c);
  for (int i = 0; i < nth; ++i) pthread_join(th[i], NULL);
  free(th);
  /* merge the label chunks' heaps of every query, descending */
  uint64_t* all = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(c.nlc * k));
  for (int64_t qi = 0; qi < nq; ++qi) {
    int64_t qb = qi / QB;
    int j = (int)(qi % QB);
    int64_t m = 0;
    for (int64_t lc = 0; lc < c.nlc; ++lc) {
      int64_t task = qb * c.nlc + lc;
      const uint64_t* h = c.heaps + ((size_t)task * QB + j) * k;
      for (int x = 0; x < c.hn[task * QB + j]; ++x) all[m++] = h[x];
    }
    qsort(all, (size_t)m, sizeof(uint64_t), cmp_key_desc);
    for (int x = 0; x < k; ++x) {
      uint64_t key = x < m ? all[x] : 0;
      if (out_keys) out_keys[qi * k + x] = key;
      if (out_ids) out_ids[qi * k + x] = key ? key_id(key) : -1;
      if (out_scores) out_scores[qi * k + x] = key ? key_score(key) : -INFINITY;
    }
  }
  free(all);
  free(c.heaps);
  free(c.hn);
}
