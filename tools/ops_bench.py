"""Measurement of the secondary rows of the hot path (SURVEY §8(a) a7 SpTTM, a8 CP-ALS, §8(f)-3
SpTTMc): GPU time through the C ABI, the roofline each is bound by, and the fp64 CPU oracle timed
beside it on a bounded sample (single thread: the oracle as it stands).  One JSON line per
(op, workload, mode, R).  Not the bench line; bench.py times the headline SpMTTKRP.

python tools/ops_bench.py [--ops ttm,ttmc,cp] [--reps 20] [--oracle-s 4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def tensor_peak_tf32():
    """Dense TF32 tensor peak (TFLOP/s): measured bf16 x the guide's nominal tf32:bf16 ratio 1/2."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("bf16_tflops", "dense_bf16_tflops", "bf16_tfs"):
            if k in d:
                return float(d[k]) * 0.5, f"measured bf16 ({k}) x 1/2"
    except Exception:
        pass
    return 2250.0 * 0.5, "fallback: nominal 2.25 PFLOP/s bf16 x 1/2"


def gpu_ms(fn, reps):
    import torch
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def oracle_rate(fn_of_sample, nnz_total, budget_s):
    """Time fn_of_sample(k) on growing prefixes until one run takes >= budget_s / 4; returns
    (nnz/s, sample nnz, seconds)."""
    k = 20000
    while True:
        k = min(k, nnz_total)
        t0 = time.perf_counter()
        fn_of_sample(k)
        dt = time.perf_counter() - t0
        if dt >= budget_s / 4 or k == nnz_total:
            return k / dt, k, dt
        k = int(k * min(8.0, max(2.0, (budget_s / 4) / max(dt, 1e-3))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="ttm,ttmc,cp")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--oracle-s", type=float, default=4.0)
    ap.add_argument("--ttmc-R", default="8,16,32")
    ap.add_argument("--ttm-layout", default="auto", choices=["auto", "fcoo", "blocked"],
                    help="auto: blocked F-COO when U does not fit the lean kernel's shared memory (32 KB)")
    ap.add_argument("--ttm-br", type=int, default=0, help="block rows of a blocked SpTTM handle (0 = default)")
    ap.add_argument("--ttm-tile", type=int, default=0, help="tile of the SpTTM handles (0 = automatic)")
    a = ap.parse_args()
    import numpy as np
    import torch

    import gen
    import oracle
    import paper_1705_09905_b200 as P
    from bench import hbm_peak
    peak, peak_src = hbm_peak()
    tpeak, tpeak_src = tensor_peak_tf32()
    ops = a.ops.split(",")

    def emit(d):
        print(json.dumps(d), flush=True)

    if "ttm" in ops:  # BASELINE configs[3]: brainq-shaped, SpTTM every mode, R=16
        w, idx, val = gen.workload("brainq")
        coo = P.Coo.from_numpy(w.dims, idx, val)
        nnz, R = int(val.shape[0]), 16
        fs = gen.factors(w.dims, R, 7)
        for n in range(3):
            blocked = a.ttm_layout == "blocked" or (a.ttm_layout == "auto" and w.dims[n] * max(4 * R, 128) > 32768)
            h = P.fcoo_build(coo, n, op=P.OP_TTM, blocked=blocked, block_rows=a.ttm_br if blocked else 0,
                             tile_nnz=a.ttm_tile)
            U = torch.from_numpy(fs[n]).cuda()
            out = torch.empty((h.info.nfib, R), device="cuda")
            ms = gpu_ms(lambda: P.fcoo_ttm(h, U, R, out), a.reps)
            ntl = h.info.ntiles
            b = nnz * 8 + (nnz + 7) // 8 + 4 * ((ntl + 31) // 32) + 4 * w.dims[n] * R + 4 * h.info.nfib * R
            rate, k, dt = oracle_rate(lambda k: oracle.ttm(w.dims, idx[:, :k], val[:k], n, fs[n]), nnz, a.oracle_s)
            emit({"op": "ttm", "workload": "brainq", "mode": n, "R": R, "tile": h.info.tile_nnz,
                  "layout": "blocked" if blocked else "fcoo", "block_rows": h.info.block_rows,
                  "nsegs": h.info.nsegs, "nfib": h.info.nfib, "ms": round(ms, 4), "gnnz_s": round(nnz / ms / 1e6, 2),
                  "gflops": round(2 * R * nnz / ms / 1e6, 1),
                  "roofline": {"bound": "hbm", "bytes": b, "achieved_gbs": round(b / ms / 1e6, 1), "peak": peak,
                               "peak_source": peak_src, "frac": round(b / ms / 1e6 / peak, 4)},
                  "cpu_oracle": {"gnnz_s": round(rate / 1e9, 5), "sample_nnz": k, "s": round(dt, 2), "cores": 1,
                                 "kind": "oracle"}})
            h.destroy()
        del coo

    if "fibre" in ops:  # Fig. 2: one nell-2 stream for SpMTTKRP on mode 0 AND SpTTM on mode 2
        w, idx, val = gen.workload("nell2")
        coo = P.Coo.from_numpy(w.dims, idx, val)
        nnz = int(val.shape[0])
        import time as _t
        for fl in (False, True):  # build cost of the second flag level
            P.fcoo_build(coo, 0, fibre_flags=fl).destroy()
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        h = P.fcoo_build(coo, 0, fibre_flags=True)
        torch.cuda.synchronize()
        b_fib = (_t.perf_counter() - t0) * 1e3
        t0 = _t.perf_counter()
        P.fcoo_build(coo, 0).destroy()
        torch.cuda.synchronize()
        b_plain = (_t.perf_counter() - t0) * 1e3
        m = h.info.prod_modes[-1]
        fs32 = [torch.from_numpy(f).cuda() for f in gen.factors(w.dims, 32, 7)]
        outm = torch.empty((w.dims[0], 32), device="cuda")
        ms_m = gpu_ms(lambda: P.fcoo_mttkrp(h, fs32, 32, outm), a.reps)
        U = torch.from_numpy(gen.factors(w.dims, 16, 7)[m]).cuda()
        outt = torch.empty((h.info.nfib, 16), device="cuda")
        ms_t = gpu_ms(lambda: P.fcoo_ttm(h, U, 16, outt), a.reps)
        t = P.fcoo_build(coo, m, op=P.OP_TTM)
        outd = torch.empty((t.info.nfib, 16), device="cuda")
        ms_d = gpu_ms(lambda: P.fcoo_ttm(t, U, 16, outd), a.reps)
        emit({"op": "fibre_level", "workload": "nell2", "handle": "MTTKRP mode 0 + FCOO_BUILD_FIBRE_FLAGS",
              "ttm_mode": m, "nfib": h.info.nfib, "build_ms_plain": round(b_plain, 2), "build_ms_fibre": round(b_fib, 2),
              "mttkrp_R32_ms": round(ms_m, 4), "ttm_R16_on_mttkrp_handle_ms": round(ms_t, 4),
              "ttm_R16_dedicated_handle_ms": round(ms_d, 4), "nnz": nnz})
        h.destroy()
        t.destroy()
        del coo

    if "ttmc" in ops or "cp" in ops:
        w, idx, val = gen.workload("nell2")
        nnz = int(val.shape[0])
        coo = P.Coo.from_numpy(w.dims, idx, val)

    if "ttmc" in ops:  # SURVEY §8(f)-3 on the nell-2-shaped tensor, every mode
        for R in [int(r) for r in a.ttmc_R.split(",")]:
            fs = gen.factors(w.dims, R, 7)
            ft = [torch.from_numpy(f).cuda() for f in fs]
            for n in range(3):
                h = P.fcoo_build(coo, n)
                W = R * R
                out = torch.empty((w.dims[n], W), device="cuda")
                ms = gpu_ms(lambda: P.fcoo_ttmc(h, ft, out), a.reps)
                useful = (2 * W + 1) * nnz  # reading Q18
                hw = 3 * 2 * W * nnz  # 3xTF32: three TF32 products per useful multiply-add
                rate, k, dt = oracle_rate(
                    lambda k: oracle.ttmc(w.dims, idx[:, :k], val[:k], n, fs, with_D=False), nnz, a.oracle_s)
                emit({"op": "ttmc", "workload": "nell2", "mode": n, "R": R, "W": W, "tile": h.info.tile_nnz,
                      "ms": round(ms, 4), "gnnz_s": round(nnz / ms / 1e6, 2),
                      "useful_tflops": round(useful / ms / 1e9, 2),
                      "roofline": {"bound": "tensor", "unit": "TFLOP/s", "achieved": round(hw / ms / 1e9, 2),
                                   "peak": tpeak, "peak_source": tpeak_src, "frac": round(hw / ms / 1e9 / tpeak, 4),
                                   "note": "mma.sync TF32 work incl. the 3x split vs the dense tf32 tcgen05 peak"},
                      "cpu_oracle": {"gnnz_s": round(rate / 1e9, 6), "useful_gflops": round(rate * (2 * W + 1) / 1e9, 3),
                                     "sample_nnz": k, "s": round(dt, 2), "cores": 1, "kind": "oracle"}})
                h.destroy()
                del out
                torch.cuda.empty_cache()

    if "cp" in ops:  # CP-ALS per iteration (Alg. 1), nell-2-shaped, R=32; oracle on a prefix sample
        R = 32
        for wl in ("nell2", "order4"):
            if wl != "nell2":
                del coo
                torch.cuda.empty_cache()
                w, idx, val = gen.workload(wl)
                nnz = int(val.shape[0])
                coo = P.Coo.from_numpy(w.dims, idx, val)
            init = gen.factors(w.dims, R, 9)

            def run(iters):
                fs_ = [torch.from_numpy(f).cuda() for f in init]
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                P.cp_als(coo, R, iters, fs_)
                torch.cuda.synchronize()
                return time.perf_counter() - t0

            run(1)
            t5 = min(run(5) for _ in range(2))
            t25 = min(run(25) for _ in range(2))
            per_iter_ms = (t25 - t5) / 20 * 1e3
            N = len(w.dims)
            k = min(nnz, 2_000_000)
            t0 = time.perf_counter()
            oracle.cp_als(w.dims, idx[:, :k], val[:k], R, 2, init)
            dt = (time.perf_counter() - t0) / 2
            emit({"op": "cp_als", "workload": wl, "R": R, "nnz": nnz, "per_iter_ms": round(per_iter_ms, 3),
                  "mttkrp_gflops_equiv": round(N * N * R * nnz / per_iter_ms / 1e6, 1),
                  "cpu_oracle": {"per_iter_s_sample": round(dt, 3), "sample_nnz": k,
                                 "per_iter_s_scaled": round(dt * nnz / k, 2), "cores": 1, "kind": "oracle",
                                 "note": "one oracle CP-ALS iteration on a draw-order prefix, scaled by nnz"}})


if __name__ == "__main__":
    main()
