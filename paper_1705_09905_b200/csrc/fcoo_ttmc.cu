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

template <int NS>
cudaError_t launch_ttmc_ns(const TtmcParams& P, cudaStream_t s) {
  const int TB = 256;
  int64_t threads = (P.tile_end - P.tile_begin) * 32;
  unsigned blocks = (unsigned)((threads + TB - 1) / TB);
  if (blocks == 0) return cudaSuccess;
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
