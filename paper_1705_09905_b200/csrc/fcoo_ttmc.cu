// fcoo_ttmc.cu — SpTTMc (Eq.(4); Table I row 3) on the F-COO engine: the same
// index-mode segments as SpMTTKRP, with the Kronecker product of the product-mode rows in place of
// their Hadamard product:
//   Y_(n)(i_n, :) = sum_{q in slice i_n} v_q * (U_a(i_a(q), :) (x) U_b(i_b(q), :)),  a < b the other
// modes in ascending mode order (Eq.(4) writes U_2(j,:) (x) U_3(k,:) for mode 1).
// Order 3 (two product modes), W = R_a * R_b <= 1024 output columns.  One warp owns one tile; lane l
// owns the W/32 consecutive output columns [l*NS, (l+1)*NS).  Fast path: when NS divides R_b, the
// lane's columns share the outer index p = l*NS / R_b and cover a contiguous run of q, so a nonzero
// costs one scalar gather of U_a(i_a, p), NS/4 float4 gathers of U_b(i_b, q0:q0+NS) and NS FFMAs.
// Segments are flushed with stores or, for the ≤ 2 tile-crossing segments, red.add (as in MTTKRP).
#include "fcoo_engine_kernels.cuh"

namespace fcoo {

namespace {

struct TtmcParams {
  const uint32_t* pa;  // indices of the outer Kronecker mode (stride nnz_pad)
  const uint32_t* pb;  // indices of the inner Kronecker mode
  const float* Ua;     // I_a x Ra
  const float* Ub;     // I_b x Rb
  int Ra, Rb, W;
  const float* val;
  const uint32_t* bf;
  const uint32_t* sf;
  const uint32_t* seg_base;
  const uint32_t* seg_coord;  // nullptr -> row = segment ordinal
  int64_t nnz, ntiles, tile_begin, tile_end;
  int T;
  float* out;  // I_n x W
};

template <int NS, bool FAST>
__global__ void __launch_bounds__(256) k_ttmc(const TtmcParams P) {
  const int lane = threadIdx.x & 31;
  const int64_t t = P.tile_begin + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (t >= P.tile_end) return;
  const int e0 = lane * NS;  // first owned column
  int pcol[NS], qcol[NS];
  bool ok[NS];
#pragma unroll
  for (int u = 0; u < NS; ++u) {
    const int e = e0 + u;
    ok[u] = e < P.W;
    pcol[u] = ok[u] ? e / P.Rb : 0;
    qcol[u] = ok[u] ? e % P.Rb : 0;
  }
  const int64_t p0 = t * (int64_t)P.T;
  const int64_t p1 = min(p0 + (int64_t)P.T, P.nnz);
  const bool left_open = !((P.sf[t >> 5] >> (t & 31)) & 1u);
  uint32_t s = P.seg_base[t] - 1u;
  uint32_t row = 0;
  if (left_open) row = P.seg_coord ? P.seg_coord[s] : s;
  bool own = false;
  float acc[NS];
#pragma unroll
  for (int u = 0; u < NS; ++u) acc[u] = 0.f;

  auto flush = [&](bool store) {
    float* o = P.out + (size_t)row * (uint32_t)P.W + e0;
#pragma unroll
    for (int u = 0; u < NS; ++u)
      if (ok[u]) {
        if (store) o[u] = acc[u];
        else atomicAdd(o + u, acc[u]);
      }
  };

  auto open_segment = [&](int64_t p) {
    if (p != p0) flush(own);
#pragma unroll
    for (int u = 0; u < NS; ++u) acc[u] = 0.f;
    own = true;
    ++s;
    row = P.seg_coord ? P.seg_coord[s] : s;
  };
  // one nonzero: gathers into registers, then NS FFMAs
  auto gather = [&](uint32_t ia, uint32_t ib, float (&ga)[FAST ? 1 : NS], float (&gb)[NS]) {
    const float* ra = P.Ua + (size_t)ia * (uint32_t)P.Ra;
    const float* rb = P.Ub + (size_t)ib * (uint32_t)P.Rb;
    if constexpr (FAST) {  // shared outer index, contiguous inner run
      ga[0] = __ldg(ra + pcol[0]);
      if constexpr (NS % 4 == 0) {
#pragma unroll
        for (int u = 0; u < NS; u += 4) {
          const float4 b = __ldg(reinterpret_cast<const float4*>(rb + qcol[0] + u));
          gb[u] = b.x; gb[u + 1] = b.y; gb[u + 2] = b.z; gb[u + 3] = b.w;
        }
      } else {
#pragma unroll
        for (int u = 0; u < NS; ++u) gb[u] = __ldg(rb + qcol[u]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < NS; ++u) {
        ga[u] = __ldg(ra + pcol[u]);
        gb[u] = __ldg(rb + qcol[u]);
      }
    }
  };
  auto accumulate = [&](float v, const float (&ga)[FAST ? 1 : NS], const float (&gb)[NS]) {
#pragma unroll
    for (int u = 0; u < NS; ++u) acc[u] = fmaf(v * ga[FAST ? 0 : u], gb[u], acc[u]);
  };

  // batches of B nonzeros: indices/values with 128-bit stream loads, every gather of the batch in
  // flight before the FMAs, segment heads tested once per batch
  constexpr int RP = FAST ? NS + 1 : 2 * NS;  // gathered registers per nonzero
  constexpr int B = RP * 8 <= 96 ? 8 : RP * 4 <= 96 ? 4 : RP * 2 <= 96 ? 2 : 1;
  const int64_t pfull = p0 + ((p1 - p0) / B) * B;
  uint32_t bfw = 0;
  for (int64_t pb = p0; pb < pfull; pb += B) {
    if (((pb - p0) & 31) == 0) bfw = ld_stream4(P.bf + (pb >> 5));
    uint32_t ia[B], ib[B], vb[B];
    ld_batch<B>(P.pa + pb, ia);
    ld_batch<B>(P.pb + pb, ib);
    ld_batch<B>(P.val + pb, vb);
    const uint32_t heads = (bfw >> ((pb - p0) & 31)) & ((1u << B) - 1u);
    float ga[B][FAST ? 1 : NS], gb[B][NS];
#pragma unroll
    for (int e = 0; e < B; ++e) gather(ia[e], ib[e], ga[e], gb[e]);
#pragma unroll
    for (int e = 0; e < B; ++e) {
      if (heads && ((heads >> e) & 1u)) open_segment(pb + e);
      accumulate(__uint_as_float(vb[e]), ga[e], gb[e]);
    }
  }
  for (int64_t p = pfull; p < p1; ++p) {  // ragged tail of the tensor's last tile
    if ((p & 31) == 0 || p == pfull) bfw = ld_stream4(P.bf + (p >> 5));
    if ((bfw >> (p & 31)) & 1u) open_segment(p);
    float ga[FAST ? 1 : NS], gb[NS];
    gather(ld_stream4(P.pa + p), ld_stream4(P.pb + p), ga, gb);
    accumulate(__uint_as_float(ld_stream4(P.val + p)), ga, gb);
  }
  const bool right_open = (t + 1 < P.ntiles) && !((P.sf[(t + 1) >> 5] >> ((t + 1) & 31)) & 1u);
  flush(own && !right_open);
}

// Staged, register-tiled variant (Ra + Rb <= kStagedMaxRow).  Per segment the output block
// Y(i_n) is the Ra x Rb matrix sum_q v_q U_a(i_a(q),:)^T U_b(i_b(q),:): a sum of rank-1 updates, so
// the warp tiles it like a GEMM accumulator.  The 32 lanes form an LP x LQ grid (LP = Ra/TP,
// LQ = Rb/TQ) and each lane owns a TP x TQ block in registers; per nonzero a lane reads TP elements
// of the staged A row and TQ elements of the staged B row (vector LDS, at most 8 distinct 16-byte
// chunks per instruction: one wavefront) and issues TP*TQ FMAs (packed FFMA2 where TQ is even).
// The warp copies each batch of kNB nonzeros' rows and values into shared memory with cp.async one
// batch ahead, and the batch's indices two batches ahead, so the L2 gather latency overlaps the
// previous batch's FMAs.  Batches never cross the tile's end: pidx and val are padded to whole
// tiles with index 0 / value 0, so a tail batch's padding adds exactly 0.
constexpr int kNB = 16;             // nonzeros per batch
constexpr int kStagedMaxRow = 128;  // Ra + Rb bound (shared memory: 2 x 16 x 129 floats per warp)
constexpr int kStagedWarps = 8;

__host__ __device__ constexpr int ttmc_rows_words(int Ra, int Rb) { return kNB * (Ra + Rb) + kNB; }
__host__ __device__ constexpr int ttmc_idx_words() { return 2 * kNB + 4; }
__host__ __device__ constexpr int ttmc_warp_words(int Ra, int Rb) {
  return 2 * ttmc_rows_words(Ra, Rb) + 2 * ttmc_idx_words();
}

// N consecutive floats from shared memory (aligned to min(16, 4N) bytes by the launch conditions)
template <int N>
__device__ __forceinline__ void lds_vec(const float* p, float (&x)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(p + i);
      x[i] = q.x; x[i + 1] = q.y; x[i + 2] = q.z; x[i + 3] = q.w;
    }
  } else if constexpr (N == 2) {
    const float2 q = *reinterpret_cast<const float2*>(p);
    x[0] = q.x; x[1] = q.y;
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = p[i];
  }
}

// RA, RB: compile-time ranks for the common square cases (0 = runtime P.Ra / P.Rb)
template <int TP, int TQ, bool V16, int RA, int RB>
__global__ void __launch_bounds__(kStagedWarps * 32) k_ttmc_staged(const TtmcParams P) {
  extern __shared__ uint4 smem_raw[];
  const int lane = threadIdx.x & 31;
  const int64_t t = P.tile_begin + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (t >= P.tile_end) return;
  const int Ra = RA ? RA : P.Ra, Rb = RB ? RB : P.Rb;
  const int RW = ttmc_rows_words(Ra, Rb);
  float* rows = reinterpret_cast<float*>(smem_raw) + (threadIdx.x / 32) * ttmc_warp_words(Ra, Rb);
  uint32_t* idxb = reinterpret_cast<uint32_t*>(rows + 2 * RW);  // 2 x {ia[NB], ib[NB], bf, pad}

  const int LQ = Rb / TQ;
  const int pa0 = (lane / LQ) * TP, qb0 = (lane % LQ) * TQ;  // the lane's block of Y(i_n)
  const int64_t p0 = t * (int64_t)P.T;
  const int64_t p1 = min(p0 + (int64_t)P.T, P.nnz);
  const int nb = (int)((p1 - p0 + kNB - 1) / kNB);
  const bool left_open = !((P.sf[t >> 5] >> (t & 31)) & 1u);
  uint32_t s = P.seg_base[t] - 1u;
  uint32_t row = 0;
  if (left_open) row = P.seg_coord ? P.seg_coord[s] : s;
  bool own = false;
  float acc[TP][TQ];
#pragma unroll
  for (int i = 0; i < TP; ++i)
#pragma unroll
    for (int j = 0; j < TQ; ++j) acc[i][j] = 0.f;
  auto flush = [&](bool store) {
    float* o = P.out + (size_t)row * (uint32_t)P.W + (uint32_t)(pa0 * Rb + qb0);
#pragma unroll
    for (int i = 0; i < TP; ++i) {
      float* oi = o + i * Rb;
      if (store) {
        if constexpr (TQ % 4 == 0) {
#pragma unroll
          for (int j = 0; j < TQ; j += 4)
            *reinterpret_cast<float4*>(oi + j) = make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < TQ; ++j) oi[j] = acc[i][j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < TQ; ++j) atomicAdd(oi + j, acc[i][j]);
      }
    }
  };
  auto open_segment = [&](int64_t p) {
    if (p != p0) flush(own);
#pragma unroll
    for (int i = 0; i < TP; ++i)
#pragma unroll
      for (int j = 0; j < TQ; ++j) acc[i][j] = 0.f;
    own = true;
    ++s;
    row = P.seg_coord ? P.seg_coord[s] : s;
  };
  // indices (and the bf word) of batch b into idx buffer b % 2
  auto issue_idx = [&](int b) {
    const int64_t pb = p0 + (int64_t)b * kNB;
    uint32_t* d = idxb + (b & 1) * ttmc_idx_words();
    if (lane < 4) cp_async16(d + lane * 4, P.pa + pb + lane * 4);
    else if (lane < 8) cp_async16(d + kNB + (lane - 4) * 4, P.pb + pb + (lane - 4) * 4);
    else if (lane == 8) cp_async4(d + 2 * kNB, P.bf + (pb >> 5));
  };
  // factor rows and values of batch b into row buffer b % 2 (indices already in shared memory)
  auto issue_rows = [&](int b) {
    const int64_t pb = p0 + (int64_t)b * kNB;
    const uint32_t* ix = idxb + (b & 1) * ttmc_idx_words();
    float* sA = rows + (b & 1) * RW;
    float* sB = sA + kNB * Ra;
    float* sV = sB + kNB * Rb;
    // chunk c = lane + 32 j of the batch's kNB * cpn chunks (cpn per nonzero: A row then B row);
    // when cpn divides 32 a lane keeps one column offset and steps 32 / cpn nonzeros per chunk
    constexpr int CW = V16 ? 4 : 1;  // words per chunk
    const int ca = Ra / CW, cpn = (Ra + Rb) / CW;
    auto copy = [&](int e, int w) {
      if (w < ca) {
        if constexpr (V16) cp_async16(sA + e * Ra + CW * w, P.Ua + (size_t)ix[e] * (uint32_t)Ra + CW * w);
        else cp_async4(sA + e * Ra + w, P.Ua + (size_t)ix[e] * (uint32_t)Ra + w);
      } else {
        const int wb = CW * (w - ca);
        if constexpr (V16) cp_async16(sB + e * Rb + wb, P.Ub + (size_t)ix[kNB + e] * (uint32_t)Rb + wb);
        else cp_async4(sB + e * Rb + wb, P.Ub + (size_t)ix[kNB + e] * (uint32_t)Rb + wb);
      }
    };
    if (32 % cpn == 0) {
      const int step = 32 / cpn, w = lane % cpn;
      for (int e = lane / cpn; e < kNB; e += step) copy(e, w);
    } else {
      for (int c = lane; c < kNB * cpn; c += 32) {
        const int e = c / cpn;
        copy(e, c - e * cpn);
      }
    }
    if constexpr (V16) {
      if (lane < kNB / 4) cp_async16(sV + lane * 4, P.val + pb + lane * 4);
    } else {
      if (lane < kNB) cp_async4(sV + lane, P.val + pb + lane);
    }
  };

  issue_idx(0);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  issue_rows(0);
  if (nb > 1) issue_idx(1);
  cp_async_commit();
  for (int b = 0; b < nb; ++b) {
    cp_async_wait<0>();  // rows of b and indices of b+1 have landed
    __syncwarp();
    const uint32_t bfw = idxb[(b & 1) * ttmc_idx_words() + 2 * kNB];
    const uint32_t heads = (bfw >> ((b * kNB) & 31)) & ((1u << kNB) - 1u);
    __syncwarp();  // every lane has read idx buffer b % 2 before issue_idx(b + 2) refills it
    if (b + 1 < nb) {
      issue_rows(b + 1);
      if (b + 2 < nb) issue_idx(b + 2);
    }
    cp_async_commit();
    const float* sA = rows + (b & 1) * RW + pa0;
    const float* sB = rows + (b & 1) * RW + kNB * Ra + qb0;
    const float* sV = rows + (b & 1) * RW + kNB * (Ra + Rb);
    // operands of nonzero e+1 are loaded before the FMAs of e (two register sets)
    float x[2][TP], y[2][TQ];
    lds_vec<TP>(sA, x[0]);
    lds_vec<TQ>(sB, y[0]);
#pragma unroll
    for (int e = 0; e < kNB; ++e) {
      const int c = e & 1;
      if (e + 1 < kNB) {
        lds_vec<TP>(sA + (e + 1) * Ra, x[c ^ 1]);
        lds_vec<TQ>(sB + (e + 1) * Rb, y[c ^ 1]);
      }
      if (heads && ((heads >> e) & 1u)) open_segment(p0 + (int64_t)b * kNB + e);
      const float v = sV[e];
#pragma unroll
      for (int i = 0; i < TP; ++i) {
        const float a = v * x[c][i];
        if constexpr (TQ % 2 == 0) {  // packed FFMA2 (same per-element rounding as fmaf)
          const float2 a2 = make_float2(a, a);
#pragma unroll
          for (int j = 0; j < TQ; j += 2) {
            const float2 r = __ffma2_rn(a2, make_float2(y[c][j], y[c][j + 1]), make_float2(acc[i][j], acc[i][j + 1]));
            acc[i][j] = r.x; acc[i][j + 1] = r.y;
          }
        } else {
#pragma unroll
          for (int j = 0; j < TQ; ++j) acc[i][j] = fmaf(a, y[c][j], acc[i][j]);
        }
      }
    }
    __syncwarp();  // row buffer b % 2 is refilled by issue_rows(b + 2)
  }
  const bool right_open = (t + 1 < P.ntiles) && !((P.sf[(t + 1) >> 5] >> ((t + 1) & 31)) & 1u);
  flush(own && !right_open);
}

template <int TP, int TQ, int RA = 0, int RB = 0>
bool try_staged(const TtmcParams& P, bool v16, cudaStream_t s, cudaError_t* err) {
  if ((RA && P.Ra != RA) || (RB && P.Rb != RB)) return false;
  // the lane grid must tile Ra x Rb exactly, and the vector LDS/STG need aligned runs
  if (P.Ra % TP || P.Rb % TQ || (P.Ra / TP) * (P.Rb / TQ) != 32) return false;
  if ((TP % 4 == 0 && P.Ra % 4) || (TP == 2 && P.Ra % 2)) return false;
  if ((TQ % 4 == 0 && P.Rb % 4) || (TQ == 2 && P.Rb % 2)) return false;
  if (TQ % 4 == 0 && (reinterpret_cast<uintptr_t>(P.out) & 15u)) return false;  // float4 stores
  const size_t smem = sizeof(float) * (size_t)kStagedWarps * ttmc_warp_words(P.Ra, P.Rb);
  const unsigned blocks = (unsigned)((P.tile_end - P.tile_begin + kStagedWarps - 1) / kStagedWarps);
  auto kern = v16 ? k_ttmc_staged<TP, TQ, true, RA, RB> : k_ttmc_staged<TP, TQ, false, RA, RB>;
  *err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (*err == cudaSuccess && blocks) {
    kern<<<blocks, kStagedWarps * 32, smem, s>>>(P);
    count_launch();
    *err = cudaGetLastError();
  }
  return true;
}

// Tensor-core variant for RA in {8, 16, 32, 64} and RB a multiple of 8: per segment Y(i_n) = A^T B with
// A(k, p) = v_k U_a(i_a(k), p) and B(k, q) = U_b(i_b(k), q), K = the segment's nonzeros, is a dense
// contraction, so each K-chunk of 8 staged nonzeros feeds mma.sync m16n8k8 TF32 tiles.  fp32
// accuracy comes from the 3xTF32 split (x = hi + lo, both TF32; A·B ≈ hi·hi + hi·lo + lo·hi,
// relative error ~2^-19 per product), and each chunk's tile product is started from zero and added
// to the fp32 register accumulator with an RN FADD, so no long accumulation chain runs inside the
// tensor core.  Staging (rows, values, indices via cp.async) is as in k_ttmc_staged, with row
// strides padded by 8 words so the fragment loads are bank-conflict free.  A segment head inside a
// chunk splits it: the sub-ranges run with the other nonzeros' values masked to 0.
// Row stride (words) of a staged factor row: a fragment load reads rows k0 + tq (tq < 4) at 8
// consecutive columns, so the stride must be 8 or 24 (mod 32) for the four rows to land on disjoint
// bank octets: R = 8 needs no padding, R = 16, 32, 64 take +8.
constexpr int mma_stride(int R) { return (R % 16 == 8) ? R : R + 8; }

// RA = 8 runs as one m16 tile whose rows 8..15 are zero (never staged, never stored).
template <int RA, int RB>
struct MmaGeom {
  static constexpr int MT = (RA + 15) / 16, NT = RB / 8;
  static constexpr int SA = mma_stride(RA), SB = mma_stride(RB);  // padded row strides (words)
  static constexpr int ROWS = kNB * (SA + SB) + kNB;  // one row buffer: A rows, B rows, values
  static constexpr int WARP = 2 * ROWS;
};

// x = hi + lo with hi = x truncated to TF32 (sign, exponent, 10 mantissa bits: one LOP3) and
// lo = x - hi exact in fp32; the tensor core reads lo's top 19 bits, so |x - hi - lo_tf32| <=
// 2^-20 |x|.  (cvt.rna.tf32.f32 lowers to a ~5-instruction sequence on sm_100a; the mask is 2.)
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int RA, int RB>
__global__ void __launch_bounds__(kStagedWarps * 32) k_ttmc_mma(const TtmcParams P) {
  using Gm = MmaGeom<RA, RB>;
  constexpr int MT = Gm::MT, NT = Gm::NT, SA = Gm::SA, SB = Gm::SB;
  extern __shared__ uint4 smem_raw[];
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;  // mma fragment coordinates
  const int64_t t = P.tile_begin + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (t >= P.tile_end) return;
  float* rows = reinterpret_cast<float*>(smem_raw) + (threadIdx.x / 32) * Gm::WARP;

  const int64_t p0 = t * (int64_t)P.T;
  const int64_t p1 = min(p0 + (int64_t)P.T, P.nnz);
  const int nb = (int)((p1 - p0 + kNB - 1) / kNB);
  const bool left_open = !((P.sf[t >> 5] >> (t & 31)) & 1u);
  uint32_t s = P.seg_base[t] - 1u;
  uint32_t row = 0;
  if (left_open) row = P.seg_coord ? P.seg_coord[s] : s;
  bool own = false;
  float acc[MT][NT][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][j][c] = 0.f;
  // C fragment (i, j): rows p = 16i + g (+8), columns q = 8j + 2tq (+1) of Y(i_n) (p outer, Eq.(4))
  auto flush = [&](bool store) {
    float* o = P.out + (size_t)row * (uint32_t)(RA * RB);
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        float* o0 = o + (16 * i + g) * RB + 8 * j + 2 * tq;
        float* o1 = o0 + 8 * RB;
        constexpr bool hi_rows = RA >= 16;  // rows 16i+g+8 exist
        if (store) {
          *reinterpret_cast<float2*>(o0) = make_float2(acc[i][j][0], acc[i][j][1]);
          if (hi_rows) *reinterpret_cast<float2*>(o1) = make_float2(acc[i][j][2], acc[i][j][3]);
        } else {
          atomicAdd(o0, acc[i][j][0]); atomicAdd(o0 + 1, acc[i][j][1]);
          if (hi_rows) { atomicAdd(o1, acc[i][j][2]); atomicAdd(o1 + 1, acc[i][j][3]); }
        }
      }
  };
  auto open_segment = [&](int64_t p) {
    if (p != p0) flush(own);
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][j][c] = 0.f;
    own = true;
    ++s;
    row = P.seg_coord ? P.seg_coord[s] : s;
  };
  // a batch's 16 + 16 indices in one register per lane (lane e < 16: i_a of nonzero e; lane
  // 16 + e: i_b of nonzero e), loaded with one coalesced 128-byte load
  auto ld_idx = [&](int b) -> uint32_t {
    const int64_t pb = p0 + (int64_t)b * kNB;
    return ld_stream4((lane < kNB ? P.pa : P.pb) + pb + (lane & (kNB - 1)));
  };
  // factor rows and values of batch b into row buffer b % 2; indices arrive by shuffle
  auto issue_rows = [&](int b, uint32_t ixr) {
    const int64_t pb = p0 + (int64_t)b * kNB;
    float* sA = rows + (b & 1) * Gm::ROWS;
    float* sB = sA + kNB * SA;
    float* sV = sB + kNB * SB;
    constexpr int CA = RA / 4, CPN = (RA + RB) / 4;  // 16-byte chunks per A row / per nonzero
    if constexpr (32 % CPN == 0) {  // a lane keeps one chunk column and steps 32/CPN nonzeros
      constexpr int STEP = 32 / CPN;
      const int w = lane % CPN;
      const bool isA = w < CA;
      const float* base = isA ? P.Ua + 4 * w : P.Ub + 4 * (w - CA);
      float* dst = isA ? sA + 4 * w : sB + 4 * (w - CA);
      const int rs = isA ? RA : RB, ds = isA ? SA : SB, src0 = isA ? 0 : kNB;
#pragma unroll
      for (int e0 = 0; e0 < kNB; e0 += STEP) {
        const int e = e0 + lane / CPN;
        const uint32_t ix = __shfl_sync(0xffffffffu, ixr, src0 + e);
        cp_async16(dst + e * ds, base + (size_t)ix * rs);
      }
    } else {
#pragma unroll
      for (int c0 = 0; c0 < kNB * CPN; c0 += 32) {
        const int c = c0 + lane;
        const int e = c / CPN, w = c - e * CPN;
        const bool isA = w < CA;
        const uint32_t ix = __shfl_sync(0xffffffffu, ixr, (isA ? 0 : kNB) + (e & (kNB - 1)));
        if (c < kNB * CPN) {
          if (isA) cp_async16(sA + e * SA + 4 * w, P.Ua + (size_t)ix * RA + 4 * w);
          else cp_async16(sB + e * SB + 4 * (w - CA), P.Ub + (size_t)ix * RB + 4 * (w - CA));
        }
      }
    }
    if (lane < kNB / 4) cp_async16(sV + lane * 4, P.val + pb + lane * 4);
  };
  // one K-chunk of 8 staged nonzeros [k0, k0+8) into d, values outside [ks, ke) masked to 0
  auto chunk = [&](float (&d)[MT][NT][4], const float* sA, const float* sB, const float* sV, int k0, int ks,
                   int ke) {
    const int ka = k0 + tq, kb = k0 + tq + 4;
    const float va = (tq >= ks && tq < ke) ? sV[ka] : 0.f;
    const float vb = (tq + 4 >= ks && tq + 4 < ke) ? sV[kb] : 0.f;
    uint32_t ah[MT][4], al[MT][4];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int m = 16 * i + g;
      split_tf32(va * sA[ka * SA + m], ah[i][0], al[i][0]);
      split_tf32(vb * sA[kb * SA + m], ah[i][2], al[i][2]);
      if constexpr (RA >= 16) {
        split_tf32(va * sA[ka * SA + m + 8], ah[i][1], al[i][1]);
        split_tf32(vb * sA[kb * SA + m + 8], ah[i][3], al[i][3]);
      } else {  // rows 8..15 of the m16 tile are padding
        ah[i][1] = al[i][1] = ah[i][3] = al[i][3] = 0u;
      }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int n = 8 * j + g;
      uint32_t bh[2], bl[2];
      split_tf32(sB[ka * SB + n], bh[0], bl[0]);
      split_tf32(sB[kb * SB + n], bh[1], bl[1]);
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        mma_tf32(d[i][j], al[i], bh);
        mma_tf32(d[i][j], ah[i], bl);
        mma_tf32(d[i][j], ah[i], bh);
      }
    }
  };
  auto add_into_acc = [&](float (&d)[MT][NT][4]) {  // fp32 RN accumulation outside the tensor core
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[i][j][c] += d[i][j][c];
          d[i][j][c] = 0.f;
        }
  };

  uint32_t ix_next = ld_idx(0);
  uint32_t bf_cur = ld_stream4(P.bf + (p0 >> 5));
  issue_rows(0, ix_next);
  cp_async_commit();
  ix_next = nb > 1 ? ld_idx(1) : 0u;
  uint32_t ix_after = nb > 2 ? ld_idx(2) : 0u;  // indices run three batches ahead of the FMAs
  for (int b = 0; b < nb; ++b) {
    const uint32_t ix_far = b + 3 < nb ? ld_idx(b + 3) : 0u;
    const uint32_t bf_next = b + 1 < nb ? ld_stream4(P.bf + ((p0 + (int64_t)(b + 1) * kNB) >> 5)) : 0u;
    if (b + 1 < nb) issue_rows(b + 1, ix_next);
    cp_async_commit();
    cp_async_wait<1>();  // rows of batch b have landed (batch b+1 stays in flight)
    __syncwarp();
    const uint32_t heads = (bf_cur >> ((b * kNB) & 31)) & ((1u << kNB) - 1u);
    const float* sA = rows + (b & 1) * Gm::ROWS;
    const float* sB = sA + kNB * SA;
    const float* sV = sB + kNB * SB;
    float d[MT][NT][4];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) d[i][j][c] = 0.f;
    if (heads == 0) {  // the common case: the whole batch continues the running segment
      chunk(d, sA, sB, sV, 0, 0, 8);
      chunk(d, sA, sB, sV, 8, 0, 8);
      add_into_acc(d);
    } else {  // sub-ranges between segment heads
#pragma unroll
      for (int k0 = 0; k0 < kNB; k0 += 8) {
        uint32_t hm = (heads >> k0) & 0xffu;
        int ks = 0;
        while (true) {
          const int e = hm ? __ffs(hm) - 1 : 8;
          if (e > ks) {
            chunk(d, sA, sB, sV, k0, ks, e);
            add_into_acc(d);
          }
          if (e == 8) break;
          open_segment(p0 + (int64_t)b * kNB + k0 + e);
          hm &= hm - 1;
          ks = e;
        }
      }
    }
    __syncwarp();  // row buffer b % 2 is refilled by issue_rows(b + 2)
    ix_next = ix_after;
    ix_after = ix_far;
    bf_cur = bf_next;
  }
  const bool right_open = (t + 1 < P.ntiles) && !((P.sf[(t + 1) >> 5] >> ((t + 1) & 31)) & 1u);
  flush(own && !right_open);
}

template <int RA, int RB>
bool try_mma(const TtmcParams& P, cudaStream_t s, cudaError_t* err) {
  if (P.Ra != RA || P.Rb != RB) return false;
  if ((reinterpret_cast<uintptr_t>(P.Ua) | reinterpret_cast<uintptr_t>(P.Ub) | reinterpret_cast<uintptr_t>(P.val) |
       reinterpret_cast<uintptr_t>(P.out)) & 15u)
    return false;
  const size_t smem = sizeof(float) * (size_t)kStagedWarps * MmaGeom<RA, RB>::WARP;
  const unsigned blocks = (unsigned)((P.tile_end - P.tile_begin + kStagedWarps - 1) / kStagedWarps);
  *err = cudaFuncSetAttribute(k_ttmc_mma<RA, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (*err == cudaSuccess && blocks) {
    k_ttmc_mma<RA, RB><<<blocks, kStagedWarps * 32, smem, s>>>(P);
    count_launch();
    *err = cudaGetLastError();
  }
  return true;
}

// Register tiles per lane, tried in order (balanced tiles first: fewest shared-memory loads).
cudaError_t launch_staged(const TtmcParams& P, bool* done, cudaStream_t s) {
  {
    cudaError_t e = cudaSuccess;
    if (try_mma<32, 32>(P, s, &e) || try_mma<16, 16>(P, s, &e) || try_mma<16, 32>(P, s, &e) ||
        try_mma<32, 16>(P, s, &e) || try_mma<16, 64>(P, s, &e) || try_mma<64, 16>(P, s, &e) ||
        try_mma<16, 8>(P, s, &e) || try_mma<32, 8>(P, s, &e) || try_mma<64, 8>(P, s, &e) ||
        try_mma<8, 8>(P, s, &e) || try_mma<8, 16>(P, s, &e) || try_mma<8, 32>(P, s, &e)) {
      *done = true;
      return e;
    }
  }
  cudaError_t e = cudaSuccess;
  const bool v16 = P.Ra % 4 == 0 && P.Rb % 4 == 0 && (reinterpret_cast<uintptr_t>(P.Ua) & 15u) == 0 &&
                   (reinterpret_cast<uintptr_t>(P.Ub) & 15u) == 0 && (reinterpret_cast<uintptr_t>(P.val) & 15u) == 0;
  *done = P.Ra + P.Rb <= kStagedMaxRow && P.W % 32 == 0 &&
          (try_staged<4, 8, 32, 32>(P, v16, s, &e) || try_staged<2, 4, 16, 16>(P, v16, s, &e) ||
           try_staged<1, 2, 8, 8>(P, v16, s, &e) || try_staged<4, 8>(P, v16, s, &e) || try_staged<8, 4>(P, v16, s, &e) || try_staged<4, 4>(P, v16, s, &e) ||
           try_staged<2, 4>(P, v16, s, &e) || try_staged<4, 2>(P, v16, s, &e) || try_staged<2, 2>(P, v16, s, &e) ||
           try_staged<1, 4>(P, v16, s, &e) || try_staged<4, 1>(P, v16, s, &e) || try_staged<1, 2>(P, v16, s, &e) ||
           try_staged<2, 1>(P, v16, s, &e) || try_staged<1, 1>(P, v16, s, &e) || try_staged<2, 8>(P, v16, s, &e) ||
           try_staged<8, 2>(P, v16, s, &e) || try_staged<1, 8>(P, v16, s, &e) || try_staged<8, 1>(P, v16, s, &e));
  return e;
}

template <int NS>
cudaError_t launch_ttmc_ns(const TtmcParams& P, cudaStream_t s) {
  const int TB = 256;
  int64_t threads = (P.tile_end - P.tile_begin) * 32;
  unsigned blocks = (unsigned)((threads + TB - 1) / TB);
  if (blocks == 0) return cudaSuccess;
  {
    bool done = false;
    cudaError_t e = launch_staged(P, &done, s);
    if (done || e != cudaSuccess) return e;
  }
  // fast path: every lane's NS columns share p and run over contiguous q (NS divides Rb); the
  // float4 form also needs 16-byte aligned runs (Rb and NS multiples of 4, aligned Ub)
  const bool fast = (P.Rb % NS == 0) && P.W % 32 == 0 &&
                    (NS % 4 != 0 || (P.Rb % 4 == 0 && (reinterpret_cast<uintptr_t>(P.Ub) & 15u) == 0));
  if (fast) k_ttmc<NS, true><<<blocks, TB, 0, s>>>(P);
  else k_ttmc<NS, false><<<blocks, TB, 0, s>>>(P);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

fcoo_status run_ttmc(fcoo_s* f, const float* const* factors, const int* ranks, float* out, cudaStream_t s) {
  Nvtx range("fcoo_ttmc");
  if (f->n_prod != 2) return fail(FCOO_ERR_ORDER, "fcoo_ttmc supports order-3 tensors (Eq.(4)); order is %d", f->order);
  // Kronecker order = ascending mode id (Eq.(4)); the handle stores product modes by extent (Q5)
  int a = 0, b = 1;
  if (f->prod_modes[0] > f->prod_modes[1]) { a = 1; b = 0; }
  const int ma = f->prod_modes[a], mb = f->prod_modes[b];
  if (!factors[ma] || !factors[mb]) return fail(FCOO_ERR_ARG, "NULL factor");
  const int Ra = ranks[ma], Rb = ranks[mb];
  if (Ra < 1 || Rb < 1 || (int64_t)Ra * Rb > 1024) return fail(FCOO_ERR_RANK, "ranks %d x %d outside [1, 1024]", Ra, Rb);
  TtmcParams P{};
  P.pa = f->pidx + (int64_t)a * f->nnz_pad;
  P.pb = f->pidx + (int64_t)b * f->nnz_pad;
  P.Ua = factors[ma];
  P.Ub = factors[mb];
  P.Ra = Ra; P.Rb = Rb; P.W = Ra * Rb;
  P.val = f->val; P.bf = f->bf; P.sf = f->sf; P.seg_base = f->seg_base;
  P.seg_coord = f->dense_rows ? nullptr : f->seg_coord;
  P.nnz = f->nnz; P.ntiles = f->ntiles; P.tile_begin = f->tile_begin; P.tile_end = f->tile_end;
  P.T = (int)f->T; P.out = out;
  FCOO_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)f->dims[f->mode] * P.W, s));
  const int ns_needed = (P.W + 31) / 32;
  cudaError_t e;
  if (ns_needed <= 1) e = launch_ttmc_ns<1>(P, s);
  else if (ns_needed <= 2) e = launch_ttmc_ns<2>(P, s);
  else if (ns_needed <= 4) e = launch_ttmc_ns<4>(P, s);
  else if (ns_needed <= 8) e = launch_ttmc_ns<8>(P, s);
  else if (ns_needed <= 16) e = launch_ttmc_ns<16>(P, s);
  else e = launch_ttmc_ns<32>(P, s);
  if (e != cudaSuccess) return fail(FCOO_ERR_CUDA, "ttmc launch: %s", cudaGetErrorString(e));
  if (f->comm) return comm_allreduce(f->comm, out, (size_t)f->dims[f->mode] * P.W, s);
  return FCOO_OK;
}

}  // namespace fcoo
