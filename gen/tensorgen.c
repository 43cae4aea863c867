/*
 * tensorgen.c — seeded synthetic INPUT generator shared by the oracle and the
 * CUDA path (the only module both sides may use).  It holds none of the
 * method's arithmetic: no sort keys, no flags, no MTTKRP/TTM/CP maths.  It only
 * draws coordinates, values and dense factor entries from a counter-based
 * generator, so every input is reproducible from (seed, stream, counter).
 *
 * Recipe:
 *   h(seed, stream, ctr) = splitmix64(splitmix64(splitmix64(seed) ^ stream) ^ ctr)
 *   mode-m coordinate of draw q: rank r ~ Zipf(alpha_m) over 1..I_m by inverse CDF
 *     (fp64 cumulative table), mapped through a seeded Fisher-Yates permutation
 *     pi_m so hot slices are scattered (alpha_m = 0 gives the uniform law).
 *   draws q = 0,1,2,... ; a coordinate tuple already drawn is skipped, until
 *     nnz distinct tuples exist ("first occurrence in draw order wins").
 *   value of draw q: (1 + (h(seed, VALUE_STREAM, q) >> 40)) * 2^-24 in (0, 1],
 *     exact in fp32.
 *   output is in draw order (unsorted) so the device sort does real work.
 *   factor entries: (h >> 40) * 2^-24 in [0,1) or (h >> 40) * 2^-23 - 1 in [-1,1).
 *
 * The dedup uses an open-addressing table with an atomic "min draw index" per
 * tuple, so the result is independent of the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TG_VALUE_STREAM 0x76616c7565ULL /* "value" */
#define TG_PERM_STREAM 0x7065726d00ULL  /* "perm" + mode */

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint64_t tg_h(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return splitmix64(splitmix64(splitmix64(seed) ^ stream) ^ ctr);
}

uint64_t tg_hash(uint64_t seed, uint64_t stream, uint64_t ctr) { return tg_h(seed, stream, ctr); }

static inline double tg_u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

/* Fill out[0..n) with counter-based uniform fp32 factor entries.
 * signed_range = 0 -> [0,1), 1 -> [-1,1).  Counter = offset + i. */
void tg_uniform_f32(uint64_t seed, uint64_t stream, int64_t offset, int64_t n, int signed_range, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t h = tg_h(seed, stream, (uint64_t)(offset + i)) >> 40; /* 24 bits */
    out[i] = signed_range ? (float)((double)h * (1.0 / 8388608.0) - 1.0) : (float)((double)h * (1.0 / 16777216.0));
  }
}

typedef struct {
  int64_t n;
  double* cdf; /* cdf[r] = sum_{t<=r} (t+1)^-alpha, r = 0..n-1 (rank r+1) */
  uint32_t* perm;
  int uniform;
} tg_mode_t;

static int tg_mode_init(tg_mode_t* md, int64_t n, double alpha, uint64_t seed, int m) {
  md->n = n;
  md->uniform = (alpha == 0.0);
  md->cdf = NULL;
  md->perm = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  if (!md->perm) return -1;
  if (!md->uniform) {
    md->cdf = (double*)malloc(sizeof(double) * (size_t)n);
    if (!md->cdf) return -1;
    double acc = 0.0;
    for (int64_t r = 0; r < n; ++r) {
      acc += pow((double)(r + 1), -alpha);
      md->cdf[r] = acc;
    }
  }
  for (int64_t i = 0; i < n; ++i) md->perm[i] = (uint32_t)i;
  for (int64_t i = n - 1; i > 0; --i) { /* seeded Fisher-Yates */
    uint64_t h = tg_h(seed, TG_PERM_STREAM + (uint64_t)m, (uint64_t)i);
    uint64_t j = (uint64_t)(((unsigned __int128)h * (unsigned __int128)(uint64_t)(i + 1)) >> 64);
    uint32_t t = md->perm[i];
    md->perm[i] = md->perm[j];
    md->perm[j] = t;
  }
  return 0;
}

static inline uint32_t tg_mode_draw(const tg_mode_t* md, uint64_t h) {
  double u = tg_u01(h);
  int64_t r;
  if (md->uniform) {
    r = (int64_t)(u * (double)md->n);
    if (r >= md->n) r = md->n - 1;
  } else {
    double target = u * md->cdf[md->n - 1];
    int64_t lo = 0, hi = md->n - 1; /* first r with cdf[r] > target */
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (md->cdf[mid] > target) hi = mid; else lo = mid + 1;
    }
    r = lo;
  }
  return md->perm[r];
}

static int bits_for(int64_t n) {
  int b = 0;
  while (b < 63 && ((int64_t)1 << b) < n) ++b;
  return b;
}

/* the dedup loop, for 64-bit and 128-bit packed tuples (tensorgen_dedup.h) */
#define TG_KEY uint64_t
#define TG_FN tg_dedup64
#define TG_HASH(k) splitmix64(k)
#define TG_LOAD(p) __atomic_load_n((p), __ATOMIC_RELAXED)
#define TG_CAS(p, e, d) __atomic_compare_exchange_n((p), (e), (d), 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)
#include "tensorgen_dedup.h"
#undef TG_KEY
#undef TG_FN
#undef TG_HASH
#undef TG_LOAD
#undef TG_CAS
typedef unsigned __int128 tg_u128;
static inline tg_u128 tg_load128(tg_u128* p) { return __sync_val_compare_and_swap(p, (tg_u128)0, (tg_u128)0); }
static inline int tg_cas128(tg_u128* p, tg_u128* expect, tg_u128 desired) {
  tg_u128 old = __sync_val_compare_and_swap(p, *expect, desired);
  if (old == *expect) return 1;
  *expect = old;
  return 0;
}
#define TG_KEY tg_u128
#define TG_FN tg_dedup128
#define TG_HASH(k) splitmix64((uint64_t)(k) ^ splitmix64((uint64_t)((k) >> 64)))
#define TG_LOAD(p) tg_load128(p)
#define TG_CAS(p, e, d) tg_cas128((p), (e), (d))
#include "tensorgen_dedup.h"
#undef TG_KEY
#undef TG_FN
#undef TG_HASH
#undef TG_LOAD
#undef TG_CAS

/*
 * Generate a duplicate-free COO tensor.
 *   idx: order*nnz uint32, SoA (idx[m*nnz + p]); val: nnz float.
 *   draws_out (may be NULL): number of draws consumed.
 * Returns 0, or -1 (alloc), -2 (bad args / nnz > prod dims), -3 (tuple > 127 bits),
 * -4 (too many duplicate draws).
 */
int tg_coo(int order, const int64_t* dims, int64_t nnz, const double* alpha, uint64_t seed,
           uint32_t* idx, float* val, int64_t* draws_out) {
  if (order < 1 || order > 8 || nnz < 0) return -2;
  int shift[8];
  int tot = 0;
  double cells = 1.0;
  for (int m = 0; m < order; ++m) {
    if (dims[m] < 1 || dims[m] > 4294967295LL) return -2;
    shift[m] = tot;
    tot += bits_for(dims[m]);
    cells *= (double)dims[m];
  }
  if (tot > 127) return -3; /* key+1 and the ~0 drop marker must stay free */
  if ((double)nnz > cells) return -2;
  if (nnz == 0) { if (draws_out) *draws_out = 0; return 0; }

  tg_mode_t md[8];
  for (int m = 0; m < order; ++m)
    if (tg_mode_init(&md[m], dims[m], alpha ? alpha[m] : 0.0, seed, m)) return -1;

  int rc;
  if (tot <= 63) rc = tg_dedup64(order, nnz, shift, tot, seed, md, idx, val, draws_out);
  else rc = tg_dedup128(order, nnz, shift, tot, seed, md, idx, val, draws_out);
  for (int m = 0; m < order; ++m) { free(md[m].cdf); free(md[m].perm); }
  return rc;
}
