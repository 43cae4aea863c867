/*
 * fcoo_oracle.cpp — plain, slow, obviously-correct fp64 CPU oracle for the F-COO
 * hot path of Liu, Wen, Sarwate, Dehnavi, "A Unified Optimization Approach for
 * Sparse Tensor Operations on GPUs" (arXiv 1705.09905).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may import, call, link or execute
 * anything under oracle/.  It shares no code, header, table or helper with the
 * CUDA library (paper_1705_09905_b200/csrc); neither includes the other.  Its
 * status codes are its own enum whose numeric values are chosen to coincide with
 * include/fcoo.h (documented there and in DESIGN.md), not included from it.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line, "S:Lnnn" = SPEC.md line,
 * "Qk" = reading k in DESIGN.md §Readings.
 *
 * Pins (tests/test_oracle_*.py, all -m "not gpu"): hand cases of S:L195-197,
 * S:L204-206; dense unfolding x explicit
 * Khatri-Rao (Eq.(5)); gradient of the CP loss; Kruskal closed form; the Fig. 3
 * TTM->Hadamard equivalence; brute-force permutations on tiny builds; CP exact
 * recovery, monotone fit, Penrose conditions, fit vs dense reconstruction.
 * No function here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <float.h>
#include <algorithm>
#include <map>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

/* Status values (same numbers as include/fcoo.h's fcoo_status, kept separate). */
enum {
  ORC_OK = 0,
  ORC_ERR_ARG = 1,
  ORC_ERR_ORDER = 2,
  ORC_ERR_MODE = 3,
  ORC_ERR_INDEX_RANGE = 4,
  ORC_ERR_DUPLICATE = 5,
  ORC_ERR_EMPTY = 6,
};

enum { ORC_OP_MTTKRP = 0, ORC_OP_TTM = 1 };

/* ------------------------------------------------------------------------- */
/* c1. Mode taxonomy, Table I and §IV-A.
 *   SpMTTKRP on mode n: index mode {n}; product modes = all others.
 *   SpTTM on mode n:    product mode {n}; index modes = all others, ascending.
 *   Q5: product modes of MTTKRP ordered by ascending extent I_m, ties by mode id.
 * Writes index modes to idx_modes[0..n_idx), product modes to prod_modes[0..n_prod). */
int orc_mode_spec_ex(int order, const int64_t* dims, int op, int mode, int desc, int* idx_modes, int* n_idx,
                     int* prod_modes, int* n_prod) {
  if (order < 2 || order > 8) return ORC_ERR_ORDER;
  if (mode < 0 || mode >= order) return ORC_ERR_MODE;
  int ni = 0, np = 0;
  if (op == ORC_OP_MTTKRP) {
    idx_modes[ni++] = mode;
    for (int m = 0; m < order; ++m)
      if (m != mode) prod_modes[np++] = m;
    /* Q5: ascending extent, ties by mode id (stable insertion sort); desc != 0: the build
     * option that orders the product modes by descending extent instead */
    for (int a = 1; a < np; ++a)
      for (int b = a; b > 0 && (desc ? dims[prod_modes[b]] > dims[prod_modes[b - 1]]
                                     : dims[prod_modes[b]] < dims[prod_modes[b - 1]]); --b)
        std::swap(prod_modes[b], prod_modes[b - 1]);
  } else if (op == ORC_OP_TTM) {
    for (int m = 0; m < order; ++m)
      if (m != mode) idx_modes[ni++] = m;
    prod_modes[np++] = mode;
  } else {
    return ORC_ERR_ARG;
  }
  *n_idx = ni;
  *n_prod = np;
  return ORC_OK;
}

int orc_mode_spec(int order, const int64_t* dims, int op, int mode, int* idx_modes, int* n_idx, int* prod_modes,
                  int* n_prod) {
  return orc_mode_spec_ex(order, dims, op, mode, 0, idx_modes, n_idx, prod_modes, n_prod);
}

/* Table II generalised to |product modes| (Q17), S:L201:
 *   core bytes = (4*|prod| + 4)*nnz + ceil(nnz/8) + 4*ceil(ceil(nnz/T)/32). */
int64_t orc_storage_bytes(int64_t nnz, int n_prod, int64_t T) {
  int64_t ntiles = (nnz + T - 1) / T;
  return (4 * (int64_t)n_prod + 4) * nnz + (nnz + 7) / 8 + 4 * ((ntiles + 31) / 32);
}

/* ------------------------------------------------------------------------- */
/* c1. F-COO build.
 *
 * Inputs: order, dims[order], nnz, idx (SoA order*nnz u32), val[nnz], op, mode, T (partition
 * length "threadlen").
 * Outputs (caller-allocated):
 *   perm[nnz]             sorted position p -> input ordinal (gather form)
 *   bf[ceil(nnz/8)]       head bit per nonzero, LSB-first bytes, pad bits 0 (Q1, Q2)
 *   sf[ceil(ntiles/32)]   sf[t] = bf[t*T], u32 words LSB-first, pad 0 (Q3)
 *   seg_base[ntiles]      number of heads in [0, t*T)
 *   seg_coord[nsegs*n_idx] index coords of the s-th head (capacity nnz*n_idx) (Q4)
 *   pidx[n_prod*nnz]      product-mode indices in sorted order (product order of Q5)
 *   pval[nnz]             values in sorted order (bitwise copies)
 *   nsegs_out
 * Returns ORC_ERR_* on invalid input: ORDER, MODE, EMPTY (nnz==0), INDEX_RANGE, DUPLICATE (Q6). */
int orc_build_ex(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int op, int mode,
                 int64_t T, int desc, uint32_t* perm, uint8_t* bf, uint32_t* sf, uint32_t* seg_base,
                 uint32_t* seg_coord, uint32_t* pidx, float* pval, int64_t* nsegs_out) {
  int idx_modes[8], prod_modes[8], n_idx = 0, n_prod = 0;
  int rc = orc_mode_spec_ex(order, dims, op, mode, desc, idx_modes, &n_idx, prod_modes, &n_prod);
  if (rc) return rc;
  if (T < 1) return ORC_ERR_ARG;
  if (nnz <= 0) return ORC_ERR_EMPTY;
  for (int m = 0; m < order; ++m)
    for (int64_t q = 0; q < nnz; ++q)
      if ((int64_t)idx[(int64_t)m * nnz + q] >= dims[m]) return ORC_ERR_INDEX_RANGE;

  /* key order: index coords (index-mode order), then product coords (product order) */
  int key_modes[8];
  for (int a = 0; a < n_idx; ++a) key_modes[a] = idx_modes[a];
  for (int a = 0; a < n_prod; ++a) key_modes[n_idx + a] = prod_modes[a];

  std::vector<int64_t> ord(nnz);
  for (int64_t q = 0; q < nnz; ++q) ord[q] = q;
  auto coord = [&](int64_t q, int a) { return idx[(int64_t)key_modes[a] * nnz + q]; };
  std::sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) {
    for (int a = 0; a < order; ++a) {
      uint32_t cx = coord(x, a), cy = coord(y, a);
      if (cx != cy) return cx < cy;
    }
    return x < y;
  });
  /* Q6: equal adjacent keys are duplicates */
  for (int64_t p = 1; p < nnz; ++p) {
    bool same = true;
    for (int a = 0; a < order && same; ++a) same = coord(ord[p], a) == coord(ord[p - 1], a);
    if (same) return ORC_ERR_DUPLICATE;
  }

  int64_t ntiles = (nnz + T - 1) / T;
  memset(bf, 0, (size_t)((nnz + 7) / 8));
  memset(sf, 0, sizeof(uint32_t) * (size_t)((ntiles + 31) / 32));
  int64_t nsegs = 0;
  for (int64_t p = 0; p < nnz; ++p) {
    perm[p] = (uint32_t)ord[p];
    /* bf[p] = 1 iff p == 0 or the index coords of perm[p] differ from perm[p-1] */
    bool head = (p == 0);
    for (int a = 0; a < n_idx && !head; ++a) head = coord(ord[p], a) != coord(ord[p - 1], a);
    if (p % T == 0) seg_base[p / T] = (uint32_t)nsegs; /* heads in [0, t*T) */
    if (head) {
      bf[p >> 3] |= (uint8_t)(1u << (p & 7));
      for (int a = 0; a < n_idx; ++a) seg_coord[nsegs * n_idx + a] = coord(ord[p], a);
      nsegs++;
      if (p % T == 0) sf[(p / T) >> 5] |= 1u << ((p / T) & 31); /* sf[t] = bf[t*T] */
    }
    for (int a = 0; a < n_prod; ++a) pidx[(int64_t)a * nnz + p] = coord(ord[p], n_idx + a);
    memcpy(&pval[p], &val[ord[p]], sizeof(float));
  }
  *nsegs_out = nsegs;
  return ORC_OK;
}

int orc_build(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int op, int mode,
              int64_t T, uint32_t* perm, uint8_t* bf, uint32_t* sf, uint32_t* seg_base, uint32_t* seg_coord,
              uint32_t* pidx, float* pval, int64_t* nsegs_out) {
  return orc_build_ex(order, dims, nnz, idx, val, op, mode, T, 0, perm, bf, sf, seg_base, seg_coord, pidx, pval,
                      nsegs_out);
}

/* ------------------------------------------------------------------------- */
/* c1b. Blocked F-COO for SpMTTKRP and SpTTM (DESIGN.md §5 "blocked layout", reading Q22).
 * The F-COO of Fig. 2 / P:L246-282 applied to the sub-tensors X_b = { nonzeros q :
 * floor(i_outer(q) / BR) == b }, b = 0, 1, ..., where "outer" is the FIRST product mode of Q5
 * (smallest extent), concatenated in b order, each padded with empty positions to a multiple of
 * T.  By linearity of Eq.(6), MTTKRP(X) = sum_b MTTKRP(X_b).  Written out:
 *   key(q) = (b(q), index coords, product coords), sorted ascending (std::sort on (key, q));
 *   block b occupies stream positions [blk_start[b], blk_start[b+1]), blk_start[0] = 0,
 *     blk_start[b+1] = blk_start[b] + ceil(n_b / T) * T  (n_b = #nonzeros of X_b; an empty block
 *     takes no positions); its real nonzeros are [blk_start[b], blk_end[b] = blk_start[b] + n_b);
 *   padding positions: perm = 0xFFFFFFFF, pidx = pk = 0, val = +0.0, bf = 0;
 *   bf[p] = 1 iff p is real and (p == blk_start[b] or the index coords differ from p-1's);
 *   sf[t] = bf[t*T]; seg_base[t] = #heads in [0, t*T); seg_coord[s] = index coords of head s;
 *   pidx[a][p] = product coord a (global index, Q5 order) of the nonzero at p;
 *   pk[p] = ((i_outer - b*BR) << IB) | i_last  with IB = ceil(log2(I_last)) (n_prod >= 2), where
 *     "last" is the last product mode of Q5; pk[p] = i_outer - b*BR when n_prod == 1.
 * SpTTM (op = TTM): the product mode is mode n, which is then also "outer" and "last" (one
 * product mode: the packed word is the local index); seg_row[s] (capacity nnz) = the ordinal of
 * blocked segment s's index tuple among all distinct tuples in lexicographic order (the fibre =
 * output row of Eq.(3)), nfib_out = the number of fibres.
 * Inputs as orc_build_ex, plus BR >= 1.  Capacities: stream arrays hold
 * nnz + nblocks*(T-1) positions (nblocks = ceil(I_outer / BR)), seg_coord nnz*n_idx.
 * Errors as orc_build_ex; ORC_ERR_ARG if the packed word does not fit in 32 bits. */
int orc_build_blocked_ex(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int op,
                         int mode, int64_t T, int64_t BR, uint32_t* perm, uint8_t* bf, uint32_t* sf,
                         uint32_t* seg_base, uint32_t* seg_coord, uint32_t* pidx, float* pval, uint32_t* pk,
                         int64_t* blk_start, int64_t* blk_end, int64_t cap, int64_t* nsegs_out,
                         int64_t* nstream_out, int64_t* nblocks_out, uint32_t* seg_row, int64_t* nfib_out) {
  int idx_modes[8], prod_modes[8], n_idx = 0, n_prod = 0;
  int rc = orc_mode_spec_ex(order, dims, op, mode, 0, idx_modes, &n_idx, prod_modes, &n_prod);
  if (rc) return rc;
  if (T < 1 || BR < 1) return ORC_ERR_ARG;
  if (nnz <= 0) return ORC_ERR_EMPTY;
  for (int m = 0; m < order; ++m)
    for (int64_t q = 0; q < nnz; ++q)
      if ((int64_t)idx[(int64_t)m * nnz + q] >= dims[m]) return ORC_ERR_INDEX_RANGE;
  const int outer = prod_modes[0], last = prod_modes[n_prod - 1];
  int IB = 0, LB = 0;
  while (((int64_t)1 << IB) < dims[last]) ++IB;
  while (((int64_t)1 << LB) < BR) ++LB;
  if (n_prod >= 2 && LB + IB > 32) return ORC_ERR_ARG;
  const int64_t nblocks = (dims[outer] + BR - 1) / BR;

  int key_modes[8];
  for (int a = 0; a < n_idx; ++a) key_modes[a] = idx_modes[a];
  for (int a = 0; a < n_prod; ++a) key_modes[n_idx + a] = prod_modes[a];
  auto coord = [&](int64_t q, int a) { return idx[(int64_t)key_modes[a] * nnz + q]; };
  auto blk = [&](int64_t q) { return (int64_t)idx[(int64_t)outer * nnz + q] / BR; };
  std::vector<int64_t> ord(nnz);
  for (int64_t q = 0; q < nnz; ++q) ord[q] = q;
  std::sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) {
    if (blk(x) != blk(y)) return blk(x) < blk(y);
    for (int a = 0; a < order; ++a) {
      uint32_t cx = coord(x, a), cy = coord(y, a);
      if (cx != cy) return cx < cy;
    }
    return x < y;
  });
  for (int64_t p = 1; p < nnz; ++p) { /* Q6 */
    bool same = true;
    for (int a = 0; a < order && same; ++a) same = coord(ord[p], a) == coord(ord[p - 1], a);
    if (same) return ORC_ERR_DUPLICATE;
  }
  /* block sizes and stream positions */
  std::vector<int64_t> nb(nblocks, 0);
  for (int64_t q = 0; q < nnz; ++q) nb[blk(q)]++;
  blk_start[0] = 0;
  for (int64_t b = 0; b < nblocks; ++b) {
    blk_end[b] = blk_start[b] + nb[b];
    blk_start[b + 1] = blk_start[b] + (nb[b] + T - 1) / T * T;
  }
  const int64_t ns = blk_start[nblocks];
  if (ns > cap) return ORC_ERR_ARG;
  const int64_t ntiles = ns / T;
  memset(bf, 0, (size_t)((ns + 7) / 8));
  memset(sf, 0, sizeof(uint32_t) * (size_t)((ntiles + 31) / 32));
  for (int64_t p = 0; p < ns; ++p) {
    perm[p] = 0xFFFFFFFFu;
    pval[p] = 0.0f;
    pk[p] = 0u;
    for (int a = 0; a < n_prod; ++a) pidx[(int64_t)a * ns + p] = 0u;
  }
  /* place the sorted nonzeros: the k-th nonzero of block b goes to blk_start[b] + k */
  std::vector<int64_t> pos_of(nnz);
  {
    int64_t k = 0;
    for (int64_t b = 0; b < nblocks; ++b)
      for (int64_t r = 0; r < nb[b]; ++r, ++k) pos_of[k] = blk_start[b] + r;
  }
  std::vector<int64_t> at(ns, -1); /* stream position -> sorted rank, -1 = padding */
  for (int64_t k = 0; k < nnz; ++k) at[pos_of[k]] = k;
  int64_t nsegs = 0;
  for (int64_t p = 0; p < ns; ++p) {
    if (p % T == 0) seg_base[p / T] = (uint32_t)nsegs;
    const int64_t k = at[p];
    if (k < 0) continue;
    const int64_t q = ord[k];
    const int64_t b = blk(q);
    bool head = (p == blk_start[b]);
    for (int a = 0; a < n_idx && !head; ++a) head = coord(q, a) != coord(ord[k - 1], a);
    if (head) {
      bf[p >> 3] |= (uint8_t)(1u << (p & 7));
      for (int a = 0; a < n_idx; ++a) seg_coord[nsegs * n_idx + a] = coord(q, a);
      nsegs++;
      if (p % T == 0) sf[(p / T) >> 5] |= 1u << ((p / T) & 31);
    }
    perm[p] = (uint32_t)q;
    for (int a = 0; a < n_prod; ++a) pidx[(int64_t)a * ns + p] = coord(q, n_idx + a);
    memcpy(&pval[p], &val[q], sizeof(float));
    const uint32_t local = (uint32_t)(idx[(int64_t)outer * nnz + q] - b * BR);
    pk[p] = n_prod >= 2 ? (uint32_t)(((uint64_t)local << IB) | idx[(int64_t)last * nnz + q]) : local;
  }
  *nsegs_out = nsegs;
  *nstream_out = ns;
  *nblocks_out = nblocks;
  /* SpTTM on a blocked stream: the output rows are the fibres of the F-COO (distinct index tuples
   * in lexicographic order); seg_row[s] = the fibre of blocked segment s */
  if (op == ORC_OP_TTM && seg_row) {
    std::map<std::vector<uint32_t>, int64_t> fib;
    for (int64_t k = 0; k < nnz; ++k) {
      std::vector<uint32_t> t(n_idx);
      for (int a = 0; a < n_idx; ++a) t[a] = coord(ord[k], a);
      fib.emplace(t, 0);
    }
    int64_t r = 0;
    for (auto& kv : fib) kv.second = r++;
    for (int64_t s2 = 0; s2 < nsegs; ++s2)
      seg_row[s2] = (uint32_t)fib.at(std::vector<uint32_t>(seg_coord + s2 * n_idx, seg_coord + (s2 + 1) * n_idx));
    *nfib_out = r;
  }
  return ORC_OK;
}

int orc_build_blocked(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int mode,
                      int64_t T, int64_t BR, uint32_t* perm, uint8_t* bf, uint32_t* sf, uint32_t* seg_base,
                      uint32_t* seg_coord, uint32_t* pidx, float* pval, uint32_t* pk, int64_t* blk_start,
                      int64_t* blk_end, int64_t cap, int64_t* nsegs_out, int64_t* nstream_out,
                      int64_t* nblocks_out) {
  return orc_build_blocked_ex(order, dims, nnz, idx, val, ORC_OP_MTTKRP, mode, T, BR, perm, bf, sf, seg_base,
                              seg_coord, pidx, pval, pk, blk_start, blk_end, cap, nsegs_out, nstream_out, nblocks_out,
                              nullptr, nullptr);
}

/* ------------------------------------------------------------------------- */
/* c2. SpMTTKRP, Eq.(5)/(6), Table I row 2, order-N (Q17):
 *   M(i_n, r) = sum_q v_q * prod_{m != n} U_m(i_m(q), r)
 * in fp64, in input order.  D(i_n, r) = sum_q |v_q * prod U| is the normaliser of
 * the acceptance metric.  U_m are fp32 row-major I_m x R (given as fp32, widened).
 * M, D: fp64 I_n x R, overwritten.  D may be NULL.
 * nthreads > 1: each thread accumulates a private M over a contiguous range of q,
 * merged in thread order (timing mode for the CPU baseline; same sum, other order). */
int orc_mttkrp(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int mode,
               const float* const* U, int R, double* M, double* D, int nthreads) {
  if (order < 2 || order > 8) return ORC_ERR_ORDER;
  if (mode < 0 || mode >= order) return ORC_ERR_MODE;
  if (R < 1) return ORC_ERR_ARG;
  int64_t In = dims[mode];
  for (int m = 0; m < order; ++m)
    for (int64_t q = 0; q < nnz; ++q)
      if ((int64_t)idx[(int64_t)m * nnz + q] >= dims[m]) return ORC_ERR_INDEX_RANGE;
  memset(M, 0, sizeof(double) * (size_t)(In * R));
  if (D) memset(D, 0, sizeof(double) * (size_t)(In * R));
  if (nthreads <= 1) {
    for (int64_t q = 0; q < nnz; ++q) {
      int64_t i = idx[(int64_t)mode * nnz + q];
      for (int r = 0; r < R; ++r) {
        double t = (double)val[q];
        for (int m = 0; m < order; ++m)
          if (m != mode) t *= (double)U[m][(int64_t)idx[(int64_t)m * nnz + q] * R + r];
        M[i * R + r] += t;
        if (D) D[i * R + r] += fabs(t);
      }
    }
    return ORC_OK;
  }
  std::vector<std::vector<double>> Mt(nthreads), Dt(nthreads);
#pragma omp parallel num_threads(nthreads)
  {
    int th = 0;
#ifdef _OPENMP
    th = omp_get_thread_num();
#endif
    Mt[th].assign((size_t)(In * R), 0.0);
    if (D) Dt[th].assign((size_t)(In * R), 0.0);
    double* Ml = Mt[th].data();
    double* Dl = D ? Dt[th].data() : nullptr;
    int64_t lo = nnz * th / nthreads, hi = nnz * (th + 1) / nthreads;
    for (int64_t q = lo; q < hi; ++q) {
      int64_t i = idx[(int64_t)mode * nnz + q];
      for (int r = 0; r < R; ++r) {
        double t = (double)val[q];
        for (int m = 0; m < order; ++m)
          if (m != mode) t *= (double)U[m][(int64_t)idx[(int64_t)m * nnz + q] * R + r];
        Ml[i * R + r] += t;
        if (Dl) Dl[i * R + r] += fabs(t);
      }
    }
  }
  for (int th = 0; th < nthreads; ++th)
    for (int64_t e = 0; e < In * R; ++e) {
      M[e] += Mt[th][e];
      if (D) D[e] += Dt[th][e];
    }
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* c3. SpTTM, Eq.(3), Table I row 1: for mode n,
 *   Y(i_{m != n}, :) += X(i) * U(i_n, :)
 * One dense R-fibre per distinct index tuple (semi-sparse output, sCOO P:L180).
 * Emitted in ascending lexicographic order of the index tuple (index modes ascending),
 * which is the F-COO segment order.  Outputs: nfib, coords[nfib*(order-1)] u32,
 * Y[nfib*R] fp64, D[nfib*R] fp64 (may be NULL).  Capacity: nnz fibres. */
int orc_ttm(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int mode,
            const float* U, int R, int64_t* nfib, uint32_t* coords, double* Y, double* D) {
  if (order < 2 || order > 8) return ORC_ERR_ORDER;
  if (mode < 0 || mode >= order) return ORC_ERR_MODE;
  if (R < 1) return ORC_ERR_ARG;
  for (int m = 0; m < order; ++m)
    for (int64_t q = 0; q < nnz; ++q)
      if ((int64_t)idx[(int64_t)m * nnz + q] >= dims[m]) return ORC_ERR_INDEX_RANGE;
  std::map<std::vector<uint32_t>, std::vector<double>> Ym, Dm;
  for (int64_t q = 0; q < nnz; ++q) {
    std::vector<uint32_t> key;
    for (int m = 0; m < order; ++m)
      if (m != mode) key.push_back(idx[(int64_t)m * nnz + q]);
    std::vector<double>& y = Ym[key];
    std::vector<double>& d = Dm[key];
    if (y.empty()) { y.assign(R, 0.0); d.assign(R, 0.0); }
    int64_t k = idx[(int64_t)mode * nnz + q];
    for (int r = 0; r < R; ++r) {
      double t = (double)val[q] * (double)U[k * R + r];
      y[r] += t;
      d[r] += fabs(t);
    }
  }
  int64_t f = 0;
  auto dit = Dm.begin();
  for (auto it = Ym.begin(); it != Ym.end(); ++it, ++dit, ++f) {
    for (int a = 0; a < order - 1; ++a) coords[f * (order - 1) + a] = it->first[a];
    for (int r = 0; r < R; ++r) {
      Y[f * R + r] = it->second[r];
      if (D) D[f * R + r] = dit->second[r];
    }
  }
  *nfib = f;
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* SpTTMc, Eq.(4), Table I row 3: for mode n,
 *   Y_(n)(i_n, :) += X(i) * (U_{m1}(i_{m1}, :) (x) U_{m2}(i_{m2}, :) (x) ...)
 * over the other modes m1 < m2 < ... in ascending mode order (Eq.(4) writes U_2(j,:) (x) U_3(k,:)
 * for mode 1; Kronecker of row vectors per Eq.(1): the first factor varies slowest).
 * U[m] is fp32 I_m x ranks[m]; Y, D: fp64 I_n x W, W = prod_{m != n} ranks[m]; D may be NULL. */
int orc_ttmc(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int mode,
             const float* const* U, const int* ranks, double* Y, double* D) {
  if (order < 2 || order > 8) return ORC_ERR_ORDER;
  if (mode < 0 || mode >= order) return ORC_ERR_MODE;
  int64_t W = 1;
  int others[8], no = 0;
  for (int m = 0; m < order; ++m)
    if (m != mode) {
      if (ranks[m] < 1) return ORC_ERR_ARG;
      others[no++] = m;
      W *= ranks[m];
    }
  for (int m = 0; m < order; ++m)
    for (int64_t q = 0; q < nnz; ++q)
      if ((int64_t)idx[(int64_t)m * nnz + q] >= dims[m]) return ORC_ERR_INDEX_RANGE;
  int64_t In = dims[mode];
  memset(Y, 0, sizeof(double) * (size_t)(In * W));
  if (D) memset(D, 0, sizeof(double) * (size_t)(In * W));
  std::vector<double> krow((size_t)W);
  for (int64_t q = 0; q < nnz; ++q) {
    /* Kronecker row: entry e = sum_a p_a * prod_{b > a} ranks[others[b]] (last factor fastest) */
    for (int64_t e = 0; e < W; ++e) {
      int64_t rem = e;
      double t = (double)val[q];
      for (int a = no - 1; a >= 0; --a) {
        int m = others[a];
        int64_t p = rem % ranks[m];
        rem /= ranks[m];
        t *= (double)U[m][(int64_t)idx[(int64_t)m * nnz + q] * ranks[m] + p];
      }
      krow[e] = t;
    }
    int64_t i = idx[(int64_t)mode * nnz + q];
    for (int64_t e = 0; e < W; ++e) {
      Y[i * W + e] += krow[e];
      if (D) D[i * W + e] += fabs(krow[e]);
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* c4. CP-ALS helpers (Alg. 1). */

/* G = A^T A for A (I x R, fp64 row-major). */
void orc_gram(int64_t I, int R, const double* A, double* G) {
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R; ++b) {
      double s = 0.0;
      for (int64_t i = 0; i < I; ++i) s += A[i * R + a] * A[i * R + b];
      G[a * R + b] = s;
    }
}

/* Moore-Penrose pseudo-inverse of a symmetric R x R matrix (the dagger of Alg. 1 line 2,
 * P:L156) by cyclic Jacobi eigendecomposition; eigenvalues <= tau = R*eps*max|lambda| are
 * treated as zero (Q14).  Returns the number of sweeps, or -1 if not symmetric. */
int orc_pinv_sym(int R, const double* G, double* P) {
  std::vector<double> A(G, G + (size_t)R * R), V((size_t)R * R, 0.0);
  double fro = 0.0;
  for (int a = 0; a < R * R; ++a) fro += G[a] * G[a];
  fro = sqrt(fro);
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R; ++b)
      if (fabs(G[a * R + b] - G[b * R + a]) > 1e-8 * (fro > 0 ? fro : 1.0)) return -1;
  for (int a = 0; a < R; ++a) V[a * R + a] = 1.0;
  int sweep = 0;
  for (; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b)
        if (a != b) off += A[a * R + b] * A[a * R + b];
    if (sqrt(off) <= 1e-15 * (fro > 0 ? fro : 1.0)) break;
    for (int p = 0; p < R - 1; ++p)
      for (int q = p + 1; q < R; ++q) {
        double apq = A[p * R + q];
        if (apq == 0.0) continue;
        double theta = (A[q * R + q] - A[p * R + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < R; ++k) { /* A <- J^T A J, rows/cols p and q */
          double akp = A[k * R + p], akq = A[k * R + q];
          A[k * R + p] = c * akp - s * akq;
          A[k * R + q] = s * akp + c * akq;
        }
        for (int k = 0; k < R; ++k) {
          double apk = A[p * R + k], aqk = A[q * R + k];
          A[p * R + k] = c * apk - s * aqk;
          A[q * R + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < R; ++k) { /* V <- V J */
          double vkp = V[k * R + p], vkq = V[k * R + q];
          V[k * R + p] = c * vkp - s * vkq;
          V[k * R + q] = s * vkp + c * vkq;
        }
      }
  }
  double lmax = 0.0;
  for (int a = 0; a < R; ++a) lmax = std::max(lmax, fabs(A[a * R + a]));
  double tau = (double)R * DBL_EPSILON * lmax;
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R; ++b) {
      double s = 0.0;
      for (int k = 0; k < R; ++k) {
        double lk = A[k * R + k];
        if (lk > tau) s += V[a * R + k] * V[b * R + k] / lk;
      }
      P[a * R + b] = s;
    }
  return sweep;
}

/* Normalise columns by their 2-norm; a zero column stays 0 with norm 0 (Alg. 1 lines 3/5/7,
 * S:L405). */
void orc_normalize(int64_t I, int R, double* A, double* lambda) {
  for (int r = 0; r < R; ++r) {
    double s = 0.0;
    for (int64_t i = 0; i < I; ++i) s += A[i * R + r] * A[i * R + r];
    s = sqrt(s);
    lambda[r] = s;
    if (s > 0)
      for (int64_t i = 0; i < I; ++i) A[i * R + r] /= s;
  }
}

/* fp64 MTTKRP with fp64 factors (used inside the CP oracle), Eq.(6) as in orc_mttkrp.
 * nthreads > 1: each thread sums a contiguous range of q into a private fp64 I_n x R array and the
 * partials are added in thread order (same sum, another association; pinned by the threads-agree
 * test).  Timing/scale only: the arithmetic per term is unchanged. */
static void mttkrp_f64(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int mode,
                       double* const* U, int R, double* M, int nthreads) {
  int64_t In = dims[mode];
  memset(M, 0, sizeof(double) * (size_t)(In * R));
  auto range = [&](int64_t q0, int64_t q1, double* out) {
    for (int64_t q = q0; q < q1; ++q) {
      int64_t i = idx[(int64_t)mode * nnz + q];
      for (int r = 0; r < R; ++r) {
        double t = (double)val[q];
        for (int m = 0; m < order; ++m)
          if (m != mode) t *= U[m][(int64_t)idx[(int64_t)m * nnz + q] * R + r];
        out[i * R + r] += t;
      }
    }
  };
  if (nthreads <= 1) {
    range(0, nnz, M);
    return;
  }
  std::vector<std::vector<double>> part((size_t)nthreads);
#pragma omp parallel num_threads(nthreads)
  {
#ifdef _OPENMP
    const int t = omp_get_thread_num();
#else
    const int t = 0;
#endif
    part[t].assign((size_t)(In * R), 0.0);
    range(nnz * t / nthreads, nnz * (t + 1) / nthreads, part[t].data());
  }
  for (int t = 0; t < nthreads; ++t)
    for (int64_t e = 0; e < In * R; ++e) M[e] += part[t][e];
}

/* CP-ALS, Algorithm 1 generalised to order N (Q9, Q13):
 *   for it in 1..iters: for n in 0..N-1:
 *     M = X_(n) (KR of the other factors)           [c2]
 *     V = Hadamard_{m != n} U_m^T U_m
 *     U_n = M V^dagger                              [orc_pinv_sym]
 *     lambda = column norms of U_n; normalise U_n  (Q13: lambda = norms of the latest factor)
 *   fit = 1 - sqrt(max(0, |X|^2 + |Xhat|^2 - 2<X,Xhat>)) / |X|  with
 *     <X,Xhat> = sum_r lambda_r sum_i M(i,r) U_N(i,r), |Xhat|^2 = lambda^T (Hadamard_m G_m) lambda
 *   stop early if tol > 0 and |fit - fit_prev| < tol ("no improvement").
 * init: order arrays of fp32 I_m x R (given).  out: factors fp64 (caller arrays), lambda[R],
 * fit_trace[iters], returns iterations done (>= 1) or -ORC_ERR_*. */
int orc_cp_als_mt(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int R,
                  int iters, double tol, const float* const* init, double* const* factors, double* lambda,
                  double* fit_trace, int nthreads) {
  if (order < 2 || order > 8) return -ORC_ERR_ORDER;
  if (R < 1 || iters < 1) return -ORC_ERR_ARG;
  if (nnz == 0) return -ORC_ERR_EMPTY;
  for (int m = 0; m < order; ++m)
    for (int64_t e = 0; e < dims[m] * R; ++e) factors[m][e] = (double)init[m][e];
  std::vector<std::vector<double>> G(order, std::vector<double>((size_t)R * R));
  /* Gram U^T U (orc_gram); nthreads > 1: per-thread partials over row ranges, added in thread
   * order (scale only, same sum) */
  auto gram_mt = [&](int64_t I, const double* A, double* Gout) {
    if (nthreads <= 1) { orc_gram(I, R, A, Gout); return; }
    std::vector<std::vector<double>> part((size_t)nthreads, std::vector<double>((size_t)R * R, 0.0));
#pragma omp parallel num_threads(nthreads)
    {
#ifdef _OPENMP
      const int t = omp_get_thread_num();
#else
      const int t = 0;
#endif
      orc_gram(I * (t + 1) / nthreads - I * t / nthreads, R, A + (I * t / nthreads) * R, part[t].data());
    }
    for (int a = 0; a < R * R; ++a) {
      double s2 = 0.0;
      for (int t = 0; t < nthreads; ++t) s2 += part[t][a];
      Gout[a] = s2;
    }
  };
  for (int m = 0; m < order; ++m) gram_mt(dims[m], factors[m], G[m].data());
  double xnorm2 = 0.0;
  for (int64_t q = 0; q < nnz; ++q) xnorm2 += (double)val[q] * (double)val[q];
  int64_t Imax = 0;
  for (int m = 0; m < order; ++m) Imax = std::max(Imax, dims[m]);
  std::vector<double> M((size_t)(Imax * R)), V((size_t)R * R), P((size_t)R * R);
  double fit_prev = 0.0;
  int it = 0;
  for (; it < iters; ++it) {
    for (int n = 0; n < order; ++n) {
      mttkrp_f64(order, dims, nnz, idx, val, n, factors, R, M.data(), nthreads);
      for (int a = 0; a < R * R; ++a) V[a] = 1.0;
      for (int m = 0; m < order; ++m)
        if (m != n)
          for (int a = 0; a < R * R; ++a) V[a] *= G[m][a];
      if (orc_pinv_sym(R, V.data(), P.data()) < 0) return -ORC_ERR_ARG;
#pragma omp parallel for num_threads(nthreads > 1 ? nthreads : 1)
      for (int64_t i = 0; i < dims[n]; ++i)
        for (int b = 0; b < R; ++b) {
          double s = 0.0;
          for (int a = 0; a < R; ++a) s += M[i * R + a] * P[a * R + b];
          factors[n][i * R + b] = s;
        }
      orc_normalize(dims[n], R, factors[n], lambda);
      gram_mt(dims[n], factors[n], G[n].data());
    }
    /* fit after the last mode; M holds MTTKRP of mode N-1 with the current other factors */
    int nl = order - 1;
    double inner = 0.0;
    for (int r = 0; r < R; ++r) {
      double s = 0.0;
      for (int64_t i = 0; i < dims[nl]; ++i) s += M[i * R + r] * factors[nl][i * R + r];
      inner += lambda[r] * s;
    }
    double xhat2 = 0.0;
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b) {
        double h = 1.0;
        for (int m = 0; m < order; ++m) h *= G[m][a * R + b];
        xhat2 += lambda[a] * lambda[b] * h;
      }
    double resid2 = xnorm2 + xhat2 - 2.0 * inner;
    double fit = 1.0 - sqrt(resid2 > 0 ? resid2 : 0.0) / sqrt(xnorm2);
    fit_trace[it] = fit;
    if (tol > 0 && it > 0 && fabs(fit - fit_prev) < tol) { ++it; break; }
    fit_prev = fit;
  }
  return it;
}

int orc_cp_als(int order, const int64_t* dims, int64_t nnz, const uint32_t* idx, const float* val, int R, int iters,
               double tol, const float* const* init, double* const* factors, double* lambda, double* fit_trace) {
  return orc_cp_als_mt(order, dims, nnz, idx, val, R, iters, tol, init, factors, lambda, fit_trace, 1);
}

} /* extern "C" */
