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

/*
 * Generate a duplicate-free COO tensor.
 *   idx: order*nnz uint32, SoA (idx[m*nnz + p]); val: nnz float.
 *   draws_out (may be NULL): number of draws consumed.
 * Returns 0, or -1 (alloc), -2 (bad args / nnz > prod dims), -3 (tuple > 63 bits),
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
  if (tot > 63) return -3; /* key+1 and the ~0 drop marker must stay free */
  if ((double)nnz > cells) return -2;
  if (nnz == 0) { if (draws_out) *draws_out = 0; return 0; }

  tg_mode_t md[8];
  for (int m = 0; m < order; ++m)
    if (tg_mode_init(&md[m], dims[m], alpha ? alpha[m] : 0.0, seed, m)) return -1;

  uint64_t cap = 1024;
  while (cap < (uint64_t)nnz * 2) cap <<= 1;
  uint64_t* tkey = (uint64_t*)malloc(sizeof(uint64_t) * cap);   /* key+1, 0 = empty */
  uint32_t* tmin = (uint32_t*)malloc(sizeof(uint32_t) * cap);   /* min draw index */
  int64_t kcap = nnz + nnz / 4 + 1024;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)kcap);
  int rc = 0;
  if (!tkey || !tmin || !keys) { rc = -1; goto done; }
  memset(tkey, 0, sizeof(uint64_t) * cap);
  memset(tmin, 0xff, sizeof(uint32_t) * cap);

  int64_t q_lo = 0, q_hi = nnz, distinct = 0;
  for (;;) {
    if (q_hi > kcap) {
      int64_t nk = q_hi + q_hi / 4;
      uint64_t* k2 = (uint64_t*)realloc(keys, sizeof(uint64_t) * (size_t)nk);
      if (!k2) { rc = -1; goto done; }
      keys = k2; kcap = nk;
    }
    if (q_hi > 4294967294LL || (double)q_hi > 64.0 * (double)nnz + 1e6) { rc = -4; goto done; }
    int rehash = 0;
    while ((uint64_t)q_hi > (cap / 10) * 7) { cap <<= 1; rehash = 1; }
    if (rehash) { /* grow the table and re-insert the draws so far (same min-q result) */
      free(tkey); free(tmin);
      tkey = (uint64_t*)malloc(sizeof(uint64_t) * cap);
      tmin = (uint32_t*)malloc(sizeof(uint32_t) * cap);
      if (!tkey || !tmin) { rc = -1; goto done; }
      memset(tkey, 0, sizeof(uint64_t) * cap);
      memset(tmin, 0xff, sizeof(uint32_t) * cap);
    }
    int64_t added = 0;
    int64_t q_from = rehash ? 0 : q_lo;
#pragma omp parallel for schedule(static) reduction(+ : added)
    for (int64_t q = q_from; q < q_hi; ++q) {
      uint64_t key = 0;
      if (q >= q_lo) {
        for (int m = 0; m < order; ++m) {
          uint32_t c = tg_mode_draw(&md[m], tg_h(seed, (uint64_t)m, (uint64_t)q));
          key |= (uint64_t)c << shift[m];
        }
        keys[q] = key;
      } else {
        key = keys[q];
      }
      uint64_t slot = splitmix64(key) & (cap - 1);
      for (;;) {
        uint64_t cur = __atomic_load_n(&tkey[slot], __ATOMIC_RELAXED);
        if (cur == 0) {
          uint64_t expect = 0;
          if (__atomic_compare_exchange_n(&tkey[slot], &expect, key + 1, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
            added++;
            break;
          }
          cur = expect;
        }
        if (cur == key + 1) break;
        slot = (slot + 1) & (cap - 1);
      }
      uint32_t qq = (uint32_t)q, old = __atomic_load_n(&tmin[slot], __ATOMIC_RELAXED);
      while (qq < old && !__atomic_compare_exchange_n(&tmin[slot], &old, qq, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
      }
    }
    distinct = rehash ? added : distinct + added;
    if (distinct >= nnz) break;
    q_lo = q_hi;
    q_hi += (nnz - distinct) + (nnz - distinct) / 4 + 16;
  }

  {
    /* survivors in draw order: draw q survives iff it is the first draw of its tuple */
    int nth = 1;
#ifdef _OPENMP
    nth = omp_get_max_threads();
#endif
    int64_t* cnt = (int64_t*)calloc((size_t)nth + 1, sizeof(int64_t));
    if (!cnt) { rc = -1; goto done; }
    int64_t total = q_hi;
#pragma omp parallel num_threads(nth)
    {
      int t = 0;
#ifdef _OPENMP
      t = omp_get_thread_num();
#endif
      int64_t lo = total * t / nth, hi = total * (t + 1) / nth, c = 0;
      for (int64_t q = lo; q < hi; ++q) {
        uint64_t key = keys[q], slot = splitmix64(key) & (cap - 1);
        while (tkey[slot] != key + 1) slot = (slot + 1) & (cap - 1);
        if (tmin[slot] == (uint32_t)q) c++; else keys[q] = ~0ULL; /* mark dropped */
      }
      cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
      for (int i = 1; i <= nth; ++i) cnt[i] += cnt[i - 1];
      int64_t pos = cnt[t];
      for (int64_t q = lo; q < hi && pos < nnz; ++q) {
        if (keys[q] == ~0ULL) continue; /* dropped duplicate */
        uint64_t key = keys[q];
        for (int m = 0; m < order; ++m) {
          int b = (m + 1 < order ? shift[m + 1] : tot) - shift[m];
          uint64_t mask = b >= 64 ? ~0ULL : (((uint64_t)1 << b) - 1);
          idx[(int64_t)m * nnz + pos] = (uint32_t)((key >> shift[m]) & mask);
        }
        val[pos] = (float)((double)(1 + (tg_h(seed, TG_VALUE_STREAM, (uint64_t)q) >> 40)) * (1.0 / 16777216.0));
        pos++;
      }
    }
    /* the last draw kept defines how many draws were consumed */
    if (draws_out) {
      int64_t seen = 0, q = 0;
      for (; q < total; ++q) if (keys[q] != ~0ULL && ++seen == nnz) break;
      *draws_out = q + 1;
    }
    free(cnt);
  }

done:
  for (int m = 0; m < order; ++m) { free(md[m].cdf); free(md[m].perm); }
  free(tkey); free(tmin); free(keys);
  return rc;
}
