/* tensorgen_dedup.h — the draw / duplicate-drop / emit loop of tg_coo, instantiated by
 * tensorgen.c for 64-bit tuple keys (tot <= 63 bits) and 128-bit keys (tot <= 127 bits).
 * Expects TG_KEY (key type), TG_FN (function name), TG_HASH(key) -> uint64_t, TG_LOAD(p) and
 * TG_CAS(p, expected_ptr, desired) (relaxed atomics on TG_KEY). */
static int TG_FN(int order, int64_t nnz, const int* shift, int tot, uint64_t seed, tg_mode_t* md,
                 uint32_t* idx, float* val, int64_t* draws_out) {
  uint64_t cap = 1024;
  while (cap < (uint64_t)nnz * 2) cap <<= 1;
  TG_KEY* tkey = (TG_KEY*)malloc(sizeof(TG_KEY) * cap);   /* key+1, 0 = empty */
  uint32_t* tmin = (uint32_t*)malloc(sizeof(uint32_t) * cap);   /* min draw index */
  int64_t kcap = nnz + nnz / 4 + 1024;
  TG_KEY* keys = (TG_KEY*)malloc(sizeof(TG_KEY) * (size_t)kcap);
  int rc = 0;
  if (!tkey || !tmin || !keys) { rc = -1; goto done; }
  memset(tkey, 0, sizeof(TG_KEY) * cap);
  memset(tmin, 0xff, sizeof(uint32_t) * cap);

  int64_t q_lo = 0, q_hi = nnz, distinct = 0;
  for (;;) {
    if (q_hi > kcap) {
      int64_t nk = q_hi + q_hi / 4;
      TG_KEY* k2 = (TG_KEY*)realloc(keys, sizeof(TG_KEY) * (size_t)nk);
      if (!k2) { rc = -1; goto done; }
      keys = k2; kcap = nk;
    }
    if (q_hi > 4294967294LL || (double)q_hi > 64.0 * (double)nnz + 1e6) { rc = -4; goto done; }
    int rehash = 0;
    while ((uint64_t)q_hi > (cap / 10) * 7) { cap <<= 1; rehash = 1; }
    if (rehash) { /* grow the table and re-insert the draws so far (same min-q result) */
      free(tkey); free(tmin);
      tkey = (TG_KEY*)malloc(sizeof(TG_KEY) * cap);
      tmin = (uint32_t*)malloc(sizeof(uint32_t) * cap);
      if (!tkey || !tmin) { rc = -1; goto done; }
      memset(tkey, 0, sizeof(TG_KEY) * cap);
      memset(tmin, 0xff, sizeof(uint32_t) * cap);
    }
    int64_t added = 0;
    int64_t q_from = rehash ? 0 : q_lo;
#pragma omp parallel for schedule(static) reduction(+ : added)
    for (int64_t q = q_from; q < q_hi; ++q) {
      TG_KEY key = 0;
      if (q >= q_lo) {
        for (int m = 0; m < order; ++m) {
          uint32_t c = tg_mode_draw(&md[m], tg_h(seed, (uint64_t)m, (uint64_t)q));
          key |= (TG_KEY)c << shift[m];
        }
        keys[q] = key;
      } else {
        key = keys[q];
      }
      uint64_t slot = TG_HASH(key) & (cap - 1);
      for (;;) {
        TG_KEY cur = TG_LOAD(&tkey[slot]);
        if (cur == 0) {
          TG_KEY expect = 0;
          if (TG_CAS(&tkey[slot], &expect, key + 1)) {
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
        TG_KEY key = keys[q];
        uint64_t slot = TG_HASH(key) & (cap - 1);
        while (tkey[slot] != key + 1) slot = (slot + 1) & (cap - 1);
        if (tmin[slot] == (uint32_t)q) c++; else keys[q] = ~(TG_KEY)0; /* mark dropped */
      }
      cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
      for (int i = 1; i <= nth; ++i) cnt[i] += cnt[i - 1];
      int64_t pos = cnt[t];
      for (int64_t q = lo; q < hi && pos < nnz; ++q) {
        if (keys[q] == ~(TG_KEY)0) continue; /* dropped duplicate */
        TG_KEY key = keys[q];
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
      for (; q < total; ++q) if (keys[q] != ~(TG_KEY)0 && ++seen == nnz) break;
      *draws_out = q + 1;
    }
    free(cnt);
  }

done:
  free(tkey); free(tmin); free(keys);
  return rc;
}
