// fcoo_cp.cu — CP-ALS (Algorithm 1) on top of the F-COO MTTKRP engine.
//
// Per mode n: MTTKRP -> M (fcoo_mttkrp, all-reduced across ranks when
// sharded); k_solve (one CTA): V = Hadamard_{m!=n} G_m, fp64 Cholesky, W = V^{-1}, falling back to
// a Jacobi pseudo-inverse when V is not positive definite (reading Q14); k_apply: U_n = M W
// (fp64 accumulation, fp32 store); k_gram_partial + k_gram_reduce: G_raw = U_n^T U_n (fp64,
// deterministic two-stage sum); k_norm_stats: lambda = sqrt(diag G_raw); k_scale: U_n /= lambda
// (reading Q13); then G_n = Gram of the stored normalised U_n.  Fast path (R | 256, R <= 64, the
// paper's ranks): k_apply_colsq (U_n = M W fused with the column norms -> lambda; only the Gram's
// diagonal was ever used) and k_gram_chunks (normalise in place + Gram partials in one pass) +
// k_gram_reduce_t (+ k_colsq_reduce): 4 launches after the MTTKRP instead of 7.  The R x R solve of mode n needs
// only the other modes' Grams, which are final before MTTKRP_n starts, so it runs on a second
// stream concurrently with the MTTKRP (the paper's "second stream") and is joined before
// k_apply.  After the last mode,
// k_inner_partial + k_fit compute the fit from <X,Xhat> = sum_r lambda_r sum_i M(i,r) U_N(i,r)
// and |Xhat|^2 = lambda^T (Hadamard G_m) lambda with no extra pass over X; the last mode's M is
// accumulated in fp64 so the cancellation in |X|^2 + |Xhat|^2 - 2<X,Xhat> near fit = 1 does
// not swamp the result.  Every reduction has a fixed order, so
// replicated ranks compute bit-identical factors from identical M.
// The paper runs the small matrix ops with CUBLAS on a second stream; here they are
// microsecond-scale single-purpose kernels, the solve on a second stream.
#include <math.h>
#include <string.h>

#include <vector>

#include "fcoo_internal.cuh"

namespace fcoo {

namespace {

constexpr int kCT = 256;  // threads per CTA for the small kernels

struct GramPtrs {
  const double* g[kMaxOrder];
};

// Deterministic block sum of a double (fixed tree).
__device__ double block_sum(double v, double* sh) {
  int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (t < w) sh[t] += sh[t + w];
    __syncthreads();
  }
  double r = sh[0];
  __syncthreads();
  return r;
}

// One CTA, R <= 48, everything in shared memory: V = Hadamard_{m != n} G_m; Cholesky V = L L^T;
// L^{-1} column-parallel by forward substitution; W = V^{-1} = L^{-T} L^{-1}.  If a pivot is not
// positive (V not positive definite) it writes status[0] = 1 and leaves W to k_solve (launched
// next with only_if_failed), which redoes the solve with the Jacobi pseudo-inverse fallback.
constexpr int kSmallR = 48;
__global__ void __launch_bounds__(kCT) k_solve_small(GramPtrs G, int order, int n, int R, double* __restrict__ W,
                                                     int* __restrict__ status) {
  __shared__ double L[kSmallR * kSmallR], Li[kSmallR * kSmallR];
  __shared__ double sh[kCT];
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x, RR = R * R;
  double tr = 0.0;
  for (int e = tid; e < RR; e += nt) {
    double v = 1.0;
    for (int m = 0; m < order; ++m)
      if (m != n) v *= G.g[m][e];
    L[e] = v;
    Li[e] = 0.0;
    if (e / R == e % R) tr += v;
  }
  if (tid == 0) fail = 0;
  tr = block_sum(tr, sh);  // (contains __syncthreads)
  const double tiny = 1e-12 * (tr > 0 ? tr / R : 1.0);
  for (int j = 0; j < R; ++j) {  // right-looking Cholesky, column j
    if (tid == 0) {
      double d = L[j * R + j];
      if (!(d > tiny)) fail = 1;
      L[j * R + j] = d > 0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    if (fail) break;
    const double ljj = L[j * R + j];
    for (int i = j + 1 + tid; i < R; i += nt) L[i * R + j] /= ljj;
    __syncthreads();
    // trailing update of the lower triangle: L[i][k] -= L[i][j] * L[k][j], j < k <= i
    for (int e = tid; e < RR; e += nt) {
      const int i = e / R, k = e % R;
      if (k > j && k <= i) L[i * R + k] -= L[i * R + j] * L[k * R + j];
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) status[0] = 1;
    return;
  }
  for (int c = tid; c < R; c += nt) {  // column c of L^{-1}
    for (int i = c; i < R; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= L[i * R + k] * Li[k * R + c];
      Li[i * R + c] = s / L[i * R + i];
    }
  }
  __syncthreads();
  for (int e = tid; e < RR; e += nt) {  // W = Li^T Li
    const int a = e / R, b = e % R;
    double s = 0.0;
    for (int k = a > b ? a : b; k < R; ++k) s += Li[k * R + a] * Li[k * R + b];
    W[e] = s;
  }
  if (tid == 0) status[0] = 0;
}

// One CTA.  V = Hadamard_{m != n} G_m; W = V^{-1} by Cholesky, else Jacobi pinv (tau = R*eps*max|lambda|).
// Scratch A, Q: R x R doubles each.  status[0] = 0 Cholesky, 1 Jacobi fallback.
// only_if_failed: return at once unless k_solve_small reported a non-positive pivot.
__global__ void k_solve(GramPtrs G, int order, int n, int R, double* __restrict__ A, double* __restrict__ Q,
                        double* __restrict__ W, int* __restrict__ status, int only_if_failed) {
  if (only_if_failed && status[0] == 0) return;
  __shared__ double sh[kCT];
  __shared__ int fail;
  __shared__ double cs[2];
  const int tid = threadIdx.x, nt = blockDim.x, RR = R * R;
  for (int e = tid; e < RR; e += nt) {
    double v = 1.0;
    for (int m = 0; m < order; ++m)
      if (m != n) v *= G.g[m][e];
    A[e] = v;   // V (kept for the fallback)
    W[e] = v;   // Cholesky works in W's lower triangle, then becomes the inverse
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  double tr = 0.0;
  for (int a = tid; a < R; a += nt) tr += A[a * R + a];
  tr = block_sum(tr, sh);
  const double tiny = 1e-12 * (tr > 0 ? tr / R : 1.0);
  // Cholesky V = L L^T in the lower triangle of W (column j at a time)
  for (int j = 0; j < R; ++j) {
    if (tid == 0) {
      double d = W[j * R + j];
      for (int k = 0; k < j; ++k) d -= W[j * R + k] * W[j * R + k];
      if (!(d > tiny)) fail = 1;
      W[j * R + j] = d > 0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    if (fail) break;
    double ljj = W[j * R + j];
    for (int i = j + 1 + tid; i < R; i += nt) {
      double s = W[i * R + j];
      for (int k = 0; k < j; ++k) s -= W[i * R + k] * W[j * R + k];
      W[i * R + j] = s / ljj;
    }
    __syncthreads();
  }
  if (!fail) {
    // inverse: column c of V^{-1} solves L L^T x = e_c; thread per column, result in Q then W
    for (int c = tid; c < R; c += nt) {
      for (int i = 0; i < R; ++i) {  // forward: L y = e_c  (y in Q[:, c])
        double s = (i == c) ? 1.0 : 0.0;
        for (int k = 0; k < i; ++k) s -= W[i * R + k] * Q[k * R + c];
        Q[i * R + c] = s / W[i * R + i];
      }
      for (int i = R - 1; i >= 0; --i) {  // backward: L^T x = y (in place in Q[:, c])
        double s = Q[i * R + c];
        for (int k = i + 1; k < R; ++k) s -= W[k * R + i] * Q[k * R + c];
        Q[i * R + c] = s / W[i * R + i];
      }
    }
    __syncthreads();
    for (int e = tid; e < RR; e += nt) W[e] = Q[e];
    if (tid == 0) status[0] = 0;
    return;
  }
  // ---- fallback: cyclic Jacobi eigendecomposition of A = V; Q accumulates eigenvectors ----
  double fro = 0.0;
  for (int e = tid; e < RR; e += nt) fro += A[e] * A[e];
  fro = sqrt(block_sum(fro, sh));
  for (int e = tid; e < RR; e += nt) Q[e] = (e / R == e % R) ? 1.0 : 0.0;
  __syncthreads();
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int e = tid; e < RR; e += nt)
      if (e / R != e % R) off += A[e] * A[e];
    off = block_sum(off, sh);
    if (sqrt(off) <= 1e-15 * (fro > 0 ? fro : 1.0)) break;
    for (int p = 0; p < R - 1; ++p)
      for (int q = p + 1; q < R; ++q) {
        if (tid == 0) {
          double apq = A[p * R + q], c = 1.0, s = 0.0;
          if (apq != 0.0) {
            double theta = (A[q * R + q] - A[p * R + p]) / (2.0 * apq);
            double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
          }
          cs[0] = c; cs[1] = s;
        }
        __syncthreads();
        double c = cs[0], s = cs[1];
        if (s != 0.0) {
          for (int k = tid; k < R; k += nt) {  // columns p, q of A and Q
            double akp = A[k * R + p], akq = A[k * R + q];
            A[k * R + p] = c * akp - s * akq;
            A[k * R + q] = s * akp + c * akq;
            double qkp = Q[k * R + p], qkq = Q[k * R + q];
            Q[k * R + p] = c * qkp - s * qkq;
            Q[k * R + q] = s * qkp + c * qkq;
          }
          __syncthreads();
          for (int k = tid; k < R; k += nt) {  // rows p, q of A
            double apk = A[p * R + k], aqk = A[q * R + k];
            A[p * R + k] = c * apk - s * aqk;
            A[q * R + k] = s * apk + c * aqk;
          }
        }
        __syncthreads();
      }
  }
  double lmax = 0.0;
  for (int a = tid; a < R; a += nt) lmax = fmax(lmax, fabs(A[a * R + a]));
  sh[tid] = lmax;
  __syncthreads();
  for (int w = nt / 2; w > 0; w >>= 1) {
    if (tid < w) sh[tid] = fmax(sh[tid], sh[tid + w]);
    __syncthreads();
  }
  const double tau = (double)R * 2.220446049250313e-16 * sh[0];
  for (int e = tid; e < RR; e += nt) {
    int a = e / R, b = e % R;
    double s = 0.0;
    for (int k = 0; k < R; ++k) {
      double lk = A[k * R + k];
      if (lk > tau) s += Q[a * R + k] * Q[b * R + k] / lk;
    }
    W[e] = s;
  }
  if (tid == 0) status[0] = 1;
}

// U[i, b] = sum_a M[i, a] W[a, b]  (fp64 accumulation)
template <class MT>
__device__ __forceinline__ double row_dot(const MT* m, const double* __restrict__ W, int R, int b) {
  double s = 0.0;
  for (int a = 0; a < R; ++a) s += (double)m[a] * W[a * R + b];
  return s;
}

// U = M W with M read from the fp32 buffer, or from the fp64 one when *use64 (fit mode gate)
__global__ void k_apply(const float* __restrict__ M, const double* __restrict__ M64, const int* __restrict__ use64,
                        const double* __restrict__ W, int64_t I, int R, float* __restrict__ U) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= I * R) return;
  int64_t i = e / R;
  int b = (int)(e % R);
  const bool f64 = use64 && *use64;
  U[e] = (float)(f64 ? row_dot(M64 + i * R, W, R, b) : row_dot(M + i * R, W, R, b));
}

// part[c][a*R+b] = sum_{i in chunk c} U[i,a] U[i,b]
__global__ void k_gram_partial(const float* __restrict__ U, int64_t I, int R, int64_t rows_per,
                               double* __restrict__ part) {
  const int c = blockIdx.x;
  const int64_t i0 = (int64_t)c * rows_per, i1 = min(I, i0 + rows_per);
  const int RR = R * R;
  for (int e = threadIdx.x; e < RR; e += blockDim.x) {
    int a = e / R, b = e % R;
    double s = 0.0;
    for (int64_t i = i0; i < i1; ++i) s += (double)U[i * R + a] * (double)U[i * R + b];
    part[(int64_t)c * RR + e] = s;
  }
}

// Fast path for R | 256, R <= 64 (the paper's ranks): U = M W over a fixed grid of row chunks,
// fused with the column sums of squares of the STORED fp32 U (the diagonal of its Gram: all that
// lambda needs, so the full pre-normalisation Gram is not formed); per-chunk partials go
// column-major to cpart for k_colsq_reduce.
__global__ void __launch_bounds__(kCT) k_apply_colsq(const float* __restrict__ M, const double* __restrict__ M64,
                                                     const int* __restrict__ use64, const double* __restrict__ W,
                                                     int64_t I, int R, float* __restrict__ U, int64_t rows_per,
                                                     double* __restrict__ cpart) {
  __shared__ double sh[kCT];
  const int tid = threadIdx.x;
  const int b = tid % R, rstep = kCT / R;
  const int64_t i0 = (int64_t)blockIdx.x * rows_per, i1 = min(I, i0 + rows_per);
  const bool f64 = use64 && *use64;
  double cs = 0.0;
  for (int64_t i = i0 + tid / R; i < i1; i += rstep) {
    const float u = (float)(f64 ? row_dot(M64 + i * R, W, R, b) : row_dot(M + i * R, W, R, b));
    U[i * R + b] = u;
    cs += (double)u * (double)u;
  }
  sh[tid] = cs;
  __syncthreads();
  if (tid < R) {
    double t = 0.0;
    for (int q = 0; q < rstep; ++q) t += sh[tid + q * R];
    cpart[(int64_t)tid * gridDim.x + blockIdx.x] = t;  // column-major: contiguous per column
  }
}

// lambda[col] = sqrt(sum_c cpart[col * nchunks + c]): one warp per column, 8 independent
// lane accumulators (memory-level parallelism), combined in a fixed order: deterministic.
__global__ void k_colsq_reduce(const double* __restrict__ cpart, int nchunks, int R, double* __restrict__ lam,
                               float* __restrict__ lam_f) {
  const int col = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (col >= R) return;
  const double* p = cpart + (int64_t)col * nchunks;
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int c = lane;
  for (; c + 7 * 32 < nchunks; c += 8 * 32) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] += p[c + k * 32];
  }
  for (int k = 0; c < nchunks; c += 32, ++k) a[k] += p[c];
  double t = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) {
    const double l = sqrt(t);
    lam[col] = l;
    if (lam_f) lam_f[col] = (float)l;
  }
}

// Gram partials for R <= 64 over a fixed grid of row chunks, written entry-major
// (part[e * nchunks + c]) for the warp-per-entry reduce.  With lam != nullptr the tile is first
// normalised exactly as k_scale does (fp32 (double)U / lambda) and written back, so the Gram is
// that of the stored normalised factor in the same pass.
template <int EPT>
__global__ void __launch_bounds__(kCT) k_gram_chunks(float* __restrict__ U, int64_t I, int R, int64_t rows_per,
                                                     const double* __restrict__ lam, double* __restrict__ part) {
  constexpr int TR = 32;
  __shared__ float tile[TR * 64];
  const int c = blockIdx.x;
  const int64_t i0 = (int64_t)c * rows_per, i1 = min(I, i0 + rows_per);
  const int RR = R * R;
  double acc[EPT];
  int ea[EPT], eb[EPT];
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    acc[k] = 0.0;
    const int e = threadIdx.x + k * kCT;
    ea[k] = e < RR ? e / R : 0;
    eb[k] = e < RR ? e % R : 0;
  }
  for (int64_t r0 = i0; r0 < i1; r0 += TR) {
    const int nr = (int)min((int64_t)TR, i1 - r0);
    __syncthreads();
    for (int q = threadIdx.x; q < nr * R; q += kCT) {
      float x = U[r0 * R + q];
      if (lam) {
        const double l = lam[q % R];
        if (l > 0) {
          x = (float)((double)x / l);
          U[r0 * R + q] = x;
        }
      }
      tile[q] = x;
    }
    __syncthreads();
    for (int r = 0; r < nr; ++r) {
#pragma unroll
      for (int k = 0; k < EPT; ++k) acc[k] += (double)tile[r * R + ea[k]] * (double)tile[r * R + eb[k]];
    }
  }
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int e = threadIdx.x + k * kCT;
    if (e < RR) part[(int64_t)e * gridDim.x + c] = acc[k];
  }
}

// G[e] = sum_c part[e * nchunks + c]: one warp per entry, lane-strided then a fixed xor tree
// (deterministic; contiguous loads).
__global__ void k_gram_reduce_t(const double* __restrict__ part, int nchunks, int RR, double* __restrict__ G) {
  const int e = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= RR) return;
  const double* p = part + (int64_t)e * nchunks;
  double t = 0.0;
  for (int c = lane; c < nchunks; c += 32) t += p[c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) G[e] = t;
}

__global__ void k_gram_reduce(const double* __restrict__ part, int nchunks, int RR, double* __restrict__ G) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= RR) return;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += part[(int64_t)c * RR + e];
  G[e] = s;
}

// lambda = column 2-norms = sqrt(diag Graw)
__global__ void k_norm_stats(const double* __restrict__ Graw, int R, double* __restrict__ lam,
                             float* __restrict__ lam_f) {
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    double l = sqrt(Graw[r * R + r]);
    lam[r] = l;
    if (lam_f) lam_f[r] = (float)l;
  }
}

__global__ void k_scale(float* __restrict__ U, int64_t I, int R, const double* __restrict__ lam) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= I * R) return;
  double l = lam[e % R];
  if (l > 0) U[e] = (float)((double)U[e] / l);
}

__global__ void k_set_int(int* p, int v0, int v1, int v2) { p[0] = v0; p[1] = v1; p[2] = v2; }

// Seeded initial factor (opts->seed != 0): U[e] = (h(seed, stream, e) >> 40) * 2^-24 with the
// counter-based h(seed, stream, ctr) = splitmix64(splitmix64(splitmix64(seed) ^ stream) ^ ctr)
// (DESIGN.md §4), i.e. 24-bit uniform values in [0, 1), exact in fp32.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_seed_uniform(float* __restrict__ U, int64_t n, uint64_t seed, uint64_t stream) {
  const uint64_t base = splitmix64(splitmix64(seed) ^ stream);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    U[e] = (float)(splitmix64(base ^ (uint64_t)e) >> 40) * (1.0f / 16777216.0f);
}

// part[c] = sum_{i in chunk c} sum_r lambda_r M[i,r] U[i,r]   (M from the fp64 buffer when *use64;
// nothing at all when run_if is given and *run_if == 0)
__global__ void k_inner_partial(const float* __restrict__ M32, const double* __restrict__ M64,
                                const int* __restrict__ use64, const int* __restrict__ run_if,
                                const float* __restrict__ U, const double* __restrict__ lam, int64_t I, int R,
                                int64_t rows_per, double* __restrict__ part) {
  __shared__ double sh[kCT];
  if (run_if && *run_if == 0) return;
  const int64_t i0 = (int64_t)blockIdx.x * rows_per, i1 = min(I, i0 + rows_per);
  const bool f64 = *use64 != 0;
  double s = 0.0;
  for (int64_t e = i0 * R + threadIdx.x; e < i1 * R; e += blockDim.x)
    s += lam[e % R] * (f64 ? M64[e] : (double)M32[e]) * (double)U[e];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_sumsq_partial(const float* __restrict__ v, int64_t n, int64_t per, double* __restrict__ part) {
  __shared__ double sh[kCT];
  const int64_t q0 = (int64_t)blockIdx.x * per, q1 = min(n, q0 + per);
  double s = 0.0;
  for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) s += (double)v[q] * (double)v[q];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// fit = 1 - sqrt(max(0, |X|^2 + |Xhat|^2 - 2 <X,Xhat>)) / |X|   (one CTA).
// Fit-precision flags g: g[0] = the last mode's main MTTKRP accumulates exact
// fp64 products (sticky); g[1] = recompute it exactly this iteration.  role 0 (main fit): if the
// main pass was fp32 and fit >= kExactFit, request the recompute.  role 1 (after the exact
// recompute; skipped unless g[1]): overwrite the fit and, if still >= kExactFit, make the next
// iterations' main pass exact.
constexpr double kExactFit = 0.9;
// The fit of iteration *itc goes to fitd[*itc] (a device counter, so one captured iteration
// replays unchanged); role 1 always advances the counter, role 0 only when inc (no role 1 launch).
__global__ void k_fit(const double* __restrict__ inner_part, int ninner, const double* __restrict__ xsq_part,
                      int nxsq, GramPtrs G, int order, const double* __restrict__ lam, int R,
                      double* __restrict__ fitd, int* __restrict__ itc, int* __restrict__ g, int role, int inc) {
  __shared__ double sh[kCT];
  if (role == 1 && g[1] == 0) {
    if (threadIdx.x == 0) ++*itc;
    return;
  }
  double inner = 0.0, xsq = 0.0, xh = 0.0;
  // fixed-order sums (thread-strided then tree): deterministic
  for (int c = threadIdx.x; c < ninner; c += blockDim.x) inner += inner_part[c];
  inner = block_sum(inner, sh);
  for (int c = threadIdx.x; c < nxsq; c += blockDim.x) xsq += xsq_part[c];
  xsq = block_sum(xsq, sh);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    double h = lam[e / R] * lam[e % R];
    for (int m = 0; m < order; ++m) h *= G.g[m][e];
    xh += h;
  }
  xh = block_sum(xh, sh);
  if (threadIdx.x == 0) {
    double r2 = xsq + xh - 2.0 * inner;
    const double fit = 1.0 - sqrt(r2 > 0 ? r2 : 0.0) / sqrt(xsq);
    fitd[*itc] = fit;
    if (role == 0) g[1] = (g[0] == 0 && fit >= kExactFit) ? 1 : 0;
    else if (fit >= kExactFit) g[0] = 1;
    if (role == 1 || inc) ++*itc;
  }
}

unsigned nblk(int64_t n, int t = kCT) { return (unsigned)((n + t - 1) / t); }

}  // namespace

fcoo_status cp_als_impl(const fcoo_coo* X, const fcoo_cp_opts* o, float* const* factors, float* lambda,
                        double* fit_trace, int* iters_done, const fcoo_allocator* alloc, cudaStream_t s) {
  if (!X || !o || !factors || !fit_trace) return fail(FCOO_ERR_ARG, "NULL argument");
  const int N = X->order, R = o->R;
  if (N < 2 || N > kMaxOrder) return fail(FCOO_ERR_ORDER, "order %d", N);
  if (R < 1 || R > 256) return fail(FCOO_ERR_RANK, "R=%d outside [1,256]", R);
  if (o->iters < 1) return fail(FCOO_ERR_ARG, "iters < 1");
  for (int m = 0; m < N; ++m) if (!factors[m]) return fail(FCOO_ERR_ARG, "factors[%d] NULL", m);
  if (iters_done) *iters_done = 0;
  Alloc al;
  if (alloc && alloc->alloc && alloc->free) { al.a = *alloc; al.custom = true; }

  // F-COO for every mode, built once up front
  std::vector<fcoo_t> H(N, nullptr);
  auto cleanup = [&]() { for (auto& h : H) { fcoo_destroy(h); h = nullptr; } };
  struct Guard { decltype(cleanup)& c; ~Guard() { c(); } } guard{cleanup};  // early returns too
  fcoo_build_opts bo{FCOO_OP_MTTKRP, o->tile_nnz > 0 ? o->tile_nnz : 0,
                     o->deterministic ? FCOO_BUILD_DETERMINISTIC : 0u, 0};
  fcoo_build_opts bb = bo;
  bb.flags |= FCOO_BUILD_BLOCKED;
  const bool try_blocked = !o->deterministic && o->layout == 0 && N <= 5;
  // dist: X is this rank's chunk; each mode's handle holds the rank's nnz-balanced rows (row shards,
  // owned-rows all-gather: fcoo_build_distributed); else tile shards of a redundant build
  const bool dist = o->dist && o->comm;
  if (o->dist && (!o->comm || o->deterministic))
    return fail(FCOO_ERR_ARG, "cp_als dist needs a comm and excludes deterministic");
  for (int n = 0; n < N; ++n) {
    fcoo_status st;
    if (dist) {
      st = try_blocked ? fcoo_build_distributed(X, n, &bb, o->comm, alloc, (void*)s, &H[n]) : FCOO_ERR_ARG;
      if (st == FCOO_ERR_ARG) st = fcoo_build_distributed(X, n, &bo, o->comm, alloc, (void*)s, &H[n]);
    } else {
      st = try_blocked ? fcoo_build(X, n, &bb, alloc, (void*)s, &H[n]) : FCOO_ERR_ARG;
      if (st == FCOO_ERR_ARG) st = fcoo_build(X, n, &bo, alloc, (void*)s, &H[n]);  // layout not applicable
    }
    if (st) { cleanup(); return st; }
    if (!dist && o->comm && o->nranks > 1) fcoo_set_shard(H[n], o->rank, o->nranks, o->comm);
    if (o->deterministic) {  // reserve the boundary partials now: nothing allocates during capture
      st = ensure_dpart(H[n], sizeof(double) * (size_t)H[n]->ntiles * 2 * (size_t)R, s);
      if (st) { cleanup(); return st; }
    }
  }
  int64_t Imax = 0;
  for (int m = 0; m < N; ++m) Imax = std::max(Imax, X->dims[m]);
  const int RR = R * R;
  // row chunks of the Gram / inner-product partial sums (<= 32 MB of fp64 partials)
  const int64_t maxchunks = std::max<int64_t>(16, std::min<int64_t>(1024, (32ll << 20) / (8ll * RR)));
  Buf M(&al, sizeof(float) * Imax * R, s), M64(&al, sizeof(double) * X->dims[N - 1] * R, s);
  Buf Gs(&al, sizeof(double) * N * RR, s), Graw(&al, sizeof(double) * RR, s);
  Buf A(&al, sizeof(double) * RR, s), Q(&al, sizeof(double) * RR, s), W(&al, sizeof(double) * RR, s);
  Buf lam(&al, sizeof(double) * R, s), part(&al, sizeof(double) * maxchunks * RR, s);
  Buf ipart(&al, sizeof(double) * maxchunks, s), xpart(&al, sizeof(double) * maxchunks, s);
  Buf fitd(&al, sizeof(double) * (o->iters + 1), s), status(&al, sizeof(int) * 2, s);
  Buf flags(&al, sizeof(int) * 3, s);  // fit-precision flags g[0], g[1] (see k_fit); g[2] = iteration
  // fast per-mode path (R | 256, R <= 64): fused apply + column norms, fused normalise + Gram
  const bool fast = (kCT % R) == 0 && R <= 64;
  constexpr int kApplyChunks = 16 * 148;  // >= one element per thread up to I*R = 9.7M
  Buf cpart(&al, sizeof(double) * kApplyChunks * R, s);
  if (!cpart.ok()) return fail(FCOO_ERR_OOM, "cp_als scratch");
  if (!M.ok() || !M64.ok() || !Gs.ok() || !Graw.ok() || !A.ok() || !Q.ok() || !W.ok() || !lam.ok() || !part.ok() || !ipart.ok() ||
      !xpart.ok() || !fitd.ok() || !status.ok() || !flags.ok()) {
    return fail(FCOO_ERR_OOM, "cp_als scratch");
  }
  // The iterations run on a private non-blocking stream joined to the caller's at both ends, so
  // they can be captured into a CUDA graph even when the caller passes the legacy default stream
  // (which cannot be captured).  The join runs before the scratch buffers are freed on `s`.
  cudaStream_t const user = s;
  struct Join {
    cudaStream_t user, ws = nullptr;
    cudaEvent_t in = nullptr, out = nullptr;
    ~Join() {
      if (!ws) return;
      cudaEventRecord(out, ws);
      cudaStreamWaitEvent(user, out, 0);
      cudaEventDestroy(in);
      cudaEventDestroy(out);
      cudaStreamDestroy(ws);  // released once its work completes
    }
  } join{user};
  if (cudaStreamCreateWithFlags(&join.ws, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&join.in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&join.out, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(join.in, user) != cudaSuccess || cudaStreamWaitEvent(join.ws, join.in, 0) != cudaSuccess) {
    if (join.ws && !join.out) { cudaStreamDestroy(join.ws); join.ws = nullptr; }
    return fail(FCOO_ERR_CUDA, "cp_als stream setup: %s", cudaGetErrorString(cudaGetLastError()));
  }
  s = join.ws;
  // second stream for the R x R solve, forked from and joined into s each mode (captured into the
  // graph as a parallel branch); high priority so its single CTA is scheduled as soon as an SM
  // slot frees up during the MTTKRP
  struct Side {
    cudaStream_t st = nullptr;
    cudaEvent_t fork = nullptr, done = nullptr;
    ~Side() {
      if (fork) cudaEventDestroy(fork);
      if (done) cudaEventDestroy(done);
      if (st) cudaStreamDestroy(st);
    }
  } side;
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&side.st, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&side.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&side.done, cudaEventDisableTiming) != cudaSuccess)
      return fail(FCOO_ERR_CUDA, "cp_als side stream: %s", cudaGetErrorString(cudaGetLastError()));
  }
  // sharded runs keep the last mode exact throughout (one fp64 all-reduce, no gated recompute)
  const bool sharded = o->comm && o->nranks > 1;
  int* g = flags.as<int>();
  int* itc = g + 2;
  k_set_int<<<1, 1, 0, s>>>(g, sharded ? 1 : 0, 0, 0);
  FCOO_LAUNCH_CHECK();
  GramPtrs gp{};
  for (int m = 0; m < N; ++m) gp.g[m] = Gs.as<double>() + (int64_t)m * RR;

  auto chunks_for = [&](int64_t I) { return (int)std::min<int64_t>(maxchunks, std::max<int64_t>(1, (I + 127) / 128)); };
  // Gram of U (R <= 64: chunked partials entry-major + warp-per-entry reduce; with lam the chunks
  // also normalise U in place first, see k_gram_chunks)
  auto gram_fast = [&](float* U, int64_t I, const double* lamp, double* out) -> fcoo_status {
    const int nc = (int)std::min<int64_t>(maxchunks, std::max<int64_t>(1, (I + 63) / 64));
    const int64_t per = (I + nc - 1) / nc;
    if (RR <= kCT) k_gram_chunks<1><<<nc, kCT, 0, s>>>(U, I, R, per, lamp, part.as<double>());
    else if (RR <= 4 * kCT) k_gram_chunks<4><<<nc, kCT, 0, s>>>(U, I, R, per, lamp, part.as<double>());
    else k_gram_chunks<16><<<nc, kCT, 0, s>>>(U, I, R, per, lamp, part.as<double>());
    FCOO_LAUNCH_CHECK();
    k_gram_reduce_t<<<nblk((int64_t)RR * 32), kCT, 0, s>>>(part.as<double>(), nc, RR, out);
    FCOO_LAUNCH_CHECK();
    return FCOO_OK;
  };
  auto gram = [&](const float* U, int64_t I, double* out) -> fcoo_status {
    if (R <= 64) return gram_fast(const_cast<float*>(U), I, nullptr, out);
    int nc = chunks_for(I);
    int64_t per = (I + nc - 1) / nc;
    k_gram_partial<<<nc, kCT, 0, s>>>(U, I, R, per, part.as<double>());
    FCOO_LAUNCH_CHECK();
    k_gram_reduce<<<nblk(RR), kCT, 0, s>>>(part.as<double>(), nc, RR, out);
    FCOO_LAUNCH_CHECK();
    return FCOO_OK;
  };
  fcoo_status st = FCOO_OK;
  if (o->seed) {  // library-seeded initial factors (stream 1000 + m, as the test generator)
    for (int m = 0; m < N; ++m) {
      const int64_t n = X->dims[m] * R;
      k_seed_uniform<<<(unsigned)std::min<int64_t>(4096, (n + kCT - 1) / kCT), kCT, 0, s>>>(factors[m], n, o->seed,
                                                                                          1000u + (uint64_t)m);
      FCOO_LAUNCH_CHECK();
    }
  }
  // initial Grams of the given factors; |X|^2
  for (int m = 0; m < N && !st; ++m) st = gram(factors[m], X->dims[m], Gs.as<double>() + (int64_t)m * RR);
  // |X|^2 partials; dist: the same number of partials on every rank, summed over the ranks
  int nx = dist ? (int)maxchunks : (int)std::min<int64_t>(maxchunks, std::max<int64_t>(1, (X->nnz + 65535) / 65536));
  int64_t xper = std::max<int64_t>(1, (X->nnz + nx - 1) / nx);
  if (!st) {
    k_sumsq_partial<<<nx, kCT, 0, s>>>(X->val, X->nnz, xper, xpart.as<double>());
    fcoo::count_launch();
    if (cudaGetLastError() != cudaSuccess) st = fail(FCOO_ERR_CUDA, "k_sumsq_partial");
    if (!st && dist) st = comm_allreduce_f64(o->comm, xpart.as<double>(), (size_t)nx, s);
  }
  // One CP-ALS iteration (Alg. 1 body), enqueued on s with no host synchronisation.
  auto iteration = [&]() -> fcoo_status {
    fcoo::Nvtx range("cp_als iteration");
    fcoo_status st = FCOO_OK;
    for (int n = 0; n < N; ++n) {
      const int64_t In = X->dims[n];
      const bool last = (n == N - 1);
      // M = MTTKRP_n.  The fit's <X, Xhat> is taken from the last mode's M, so near fit 1 that
      // one accumulates exact fp64 products: both launches are enqueued and
      // the device flag g[0] lets exactly one of them work, with no host synchronisation.
      // fork: the solve for mode n reads only G_m (m != n), final at this point
      FCOO_CUDA_TRY(cudaEventRecord(side.fork, s));
      FCOO_CUDA_TRY(cudaStreamWaitEvent(side.st, side.fork, 0));
      if (R <= kSmallR) {
        k_solve_small<<<1, kCT, 0, side.st>>>(gp, N, n, R, W.as<double>(), status.as<int>());
        FCOO_LAUNCH_CHECK();
      }
      k_solve<<<1, kCT, 0, side.st>>>(gp, N, n, R, A.as<double>(), Q.as<double>(), W.as<double>(),
                                      status.as<int>(), R <= kSmallR ? 1 : 0);
      FCOO_LAUNCH_CHECK();
      FCOO_CUDA_TRY(cudaEventRecord(side.done, side.st));
      if (last && sharded) {
        st = run_mttkrp_f64(H[n], factors, R, M64.as<double>(), s);
        if (!st && H[n]->row_comm)  // row shards: each rank's rows are complete
          st = comm_gather_rows_f64(H[n]->row_comm, M64.as<double>(), H[n]->row_bounds, R, s);
        else if (!st)
          st = comm_allreduce_f64(o->comm, M64.as<double>(), (size_t)In * R, s);
      } else if (last) {
        st = run_mttkrp(H[n], factors, R, M.as<float>(), s, g, 0);
        if (!st) st = run_mttkrp_f64(H[n], factors, R, M64.as<double>(), s, g, 1);
      } else {
        st = fcoo_mttkrp(H[n], factors, R, M.as<float>(), (void*)s);
      }
      if (st) return st;
      FCOO_CUDA_TRY(cudaStreamWaitEvent(s, side.done, 0));  // join: W ready
      if (fast) {
        const int nb = (int)std::min<int64_t>(kApplyChunks, std::max<int64_t>(1, (In * R + kCT - 1) / kCT));
        const int64_t per = (In + nb - 1) / nb;
        k_apply_colsq<<<nb, kCT, 0, s>>>(M.as<float>(), M64.as<double>(), last ? g : nullptr, W.as<double>(), In, R,
                                         factors[n], per, cpart.as<double>());
        FCOO_LAUNCH_CHECK();
        k_colsq_reduce<<<nblk((int64_t)R * 32), kCT, 0, s>>>(cpart.as<double>(), nb, R, lam.as<double>(), lambda);
        FCOO_LAUNCH_CHECK();
        // normalise in place and take the Gram of the STORED (normalised, fp32) factor in the same
        // pass, so |Xhat|^2 and V describe exactly the model held in memory
        st = gram_fast(factors[n], In, lam.as<double>(), Gs.as<double>() + (int64_t)n * RR);
        if (st) return st;
        continue;
      }
      k_apply<<<nblk(In * R), kCT, 0, s>>>(M.as<float>(), M64.as<double>(), last ? g : nullptr, W.as<double>(),
                                           In, R, factors[n]);
      FCOO_LAUNCH_CHECK();
      st = gram(factors[n], In, Graw.as<double>());
      if (st) return st;
      k_norm_stats<<<1, kCT, 0, s>>>(Graw.as<double>(), R, lam.as<double>(), lambda);
      FCOO_LAUNCH_CHECK();
      k_scale<<<nblk(In * R), kCT, 0, s>>>(factors[n], In, R, lam.as<double>());
      FCOO_LAUNCH_CHECK();
      // Gram of the STORED (normalised, fp32) factor, so |Xhat|^2 and V describe exactly the
      // model held in memory
      st = gram(factors[n], In, Gs.as<double>() + (int64_t)n * RR);
      if (st) return st;
    }
    const int nl = N - 1;
    const int64_t Il = X->dims[nl];
    int nc = chunks_for(Il);
    int64_t per = (Il + nc - 1) / nc;
    k_inner_partial<<<nc, kCT, 0, s>>>(M.as<float>(), M64.as<double>(), g, nullptr, factors[nl],
                                       lam.as<double>(), Il, R, per, ipart.as<double>());
    FCOO_LAUNCH_CHECK();
    k_fit<<<1, kCT, 0, s>>>(ipart.as<double>(), nc, xpart.as<double>(), nx, gp, N, lam.as<double>(), R,
                            fitd.as<double>(), itc, g, 0, sharded ? 1 : 0);
    FCOO_LAUNCH_CHECK();
    if (!sharded) {
      // the fp32 fit reached kExactFit: recompute the last mode's M exactly (it depends only on
      // the other modes' factors, unchanged since) and take the fit again -- all gated on g[1]
      st = run_mttkrp_f64(H[nl], factors, R, M64.as<double>(), s, g + 1, 1);
      if (st) return st;
      k_inner_partial<<<nc, kCT, 0, s>>>(M.as<float>(), M64.as<double>(), g + 1, g + 1, factors[nl],
                                         lam.as<double>(), Il, R, per, ipart.as<double>());
      FCOO_LAUNCH_CHECK();
      k_fit<<<1, kCT, 0, s>>>(ipart.as<double>(), nc, xpart.as<double>(), nx, gp, N, lam.as<double>(), R,
                              fitd.as<double>(), itc, g, 1, 0);
      FCOO_LAUNCH_CHECK();
    }
    return FCOO_OK;
  };

  // Iteration 0 runs eagerly; iteration 1 is captured into a CUDA graph and every later iteration
  // replays it (the ~45 small launches of an iteration become one graph launch).  Any capture or
  // instantiation failure falls back to eager launches.
  cudaGraphExec_t exec = nullptr;
  uint64_t graph_kernels = 0;
  struct ExecGuard { cudaGraphExec_t& e; ~ExecGuard() { if (e) cudaGraphExecDestroy(e); } } exec_guard{exec};
  double fit_prev = 0.0;
  int it = 0;
  for (; it < o->iters && !st; ++it) {
    if (it == 1 && o->iters > 2 &&
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      const uint64_t before = fcoo::g_launches.load();
      fcoo_status cst = iteration();
      const uint64_t captured = fcoo::g_launches.load() - before;
      fcoo::g_launches.fetch_sub(captured);  // recorded, not executed
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamEndCapture(s, &graph);
      if (cst) {  // something refused to be captured: run this and every later iteration eagerly
        if (graph) cudaGraphDestroy(graph);
        graph = nullptr;
        ce = cudaErrorStreamCaptureInvalidated;
      }
      if (ce == cudaSuccess && graph) {
        size_t nn = 0;
        cudaGraphGetNodes(graph, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
        for (auto nd : nodes) {
          cudaGraphNodeType ty;
          if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++graph_kernels;
        }
        if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) exec = nullptr;
        cudaGraphDestroy(graph);
      }
      if (!exec) (void)cudaGetLastError();  // eager fallback below
    } else if (it == 1) {
      (void)cudaGetLastError();  // a refused capture must not leave a sticky error behind
    }
    if (exec) {
      cudaError_t ce = cudaGraphLaunch(exec, s);
      if (ce != cudaSuccess) { st = fail(FCOO_ERR_CUDA, "graph launch: %s", cudaGetErrorString(ce)); break; }
      fcoo::count_launch(graph_kernels);
    } else {
      st = iteration();
      if (st) break;
    }
    if (iters_done) *iters_done = it + 1;
    if (o->tol > 0) {  // the stopping rule needs the fit on the host every iteration
      double fit = 0.0;
      cudaError_t ce = cudaMemcpyAsync(&fit, fitd.as<double>() + it, sizeof(double), cudaMemcpyDeviceToHost, s);
      if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
      if (ce != cudaSuccess) { st = fail(FCOO_ERR_CUDA, "fit readback: %s", cudaGetErrorString(ce)); break; }
      if (it > 0 && fabs(fit - fit_prev) < o->tol) { ++it; break; }
      fit_prev = fit;
    }
  }
  if (!st && it > 0) {  // fit trace (one readback when tol == 0)
    cudaError_t ce = cudaMemcpyAsync(fit_trace, fitd.p, sizeof(double) * it, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) st = fail(FCOO_ERR_CUDA, "fit readback: %s", cudaGetErrorString(ce));
  }
  // the handles are freed stream-ordered on the caller's stream: every kernel enqueued on the
  // private and side streams must be ordered before that (also on the error paths)
  cudaEventRecord(side.done, side.st);
  cudaStreamWaitEvent(s, side.done, 0);
  cudaEventRecord(join.out, s);
  cudaStreamWaitEvent(user, join.out, 0);
  cleanup();
  return st;
}

}  // namespace fcoo

extern "C" fcoo_status cp_als(const fcoo_coo* tensor, const fcoo_cp_opts* opts, float* const* factors, float* lambda,
                              double* fit_trace, int* iters_done, const fcoo_allocator* alloc, void* stream) {
  return fcoo::cp_als_impl(tensor, opts, factors, lambda, fit_trace, iters_done, alloc, (cudaStream_t)stream);
}
