"""Quick per-(R, mode) timing sweep of fcoo_mttkrp on a workload (engine A/B experiments).

python tools/sweep.py [--workload nell2] [--R 16,32,64] [--tile 256] [--layout blocked|fcoo]
Prints one JSON line per (R, mode): ms (CUDA events, 10 reps after 2 warm-up), G nnz/s, %HBM.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="nell2")
    ap.add_argument("--R", default="16,32,64")
    ap.add_argument("--tile", type=int, default=0, help="0 = automatic")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--op", default="mttkrp")
    ap.add_argument("--desc", action="store_true", help="FCOO_BUILD_PRODUCT_DESC")
    ap.add_argument("--layout", default="fcoo", choices=["fcoo", "blocked"], help="MTTKRP handle layout")
    ap.add_argument("--flush", action="store_true",
                    help="SURVEY 8(d) protocol: write a 2 x L2 scratch buffer before every rep (cold factors and "
                         "stream), time each rep alone, report median and min")
    a = ap.parse_args()
    import torch

    import gen
    import paper_1705_09905_b200 as P
    from bench import compulsory_bytes, hbm_peak
    w, idx, val = gen.workload(a.workload)
    coo = P.Coo.from_numpy(w.dims, idx, val)
    N = len(w.dims)
    nnz = val.shape[0]
    peak, _ = hbm_peak()
    import time
    for n in range(N):
        bop = P.OP_TTM if a.op == "ttm" else P.OP_MTTKRP
        blk = a.layout == "blocked" and bop == P.OP_MTTKRP
        P.fcoo_build(coo, n, op=bop, tile_nnz=a.tile, product_desc=a.desc, blocked=blk).destroy()  # warm allocator / CUB
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = P.fcoo_build(coo, n, op=bop, tile_nnz=a.tile, product_desc=a.desc, blocked=blk)
        torch.cuda.synchronize()
        build_ms = (time.perf_counter() - t0) * 1e3
        for R in [int(x) for x in a.R.split(",")]:
            fs = [torch.from_numpy(f).cuda() for f in gen.factors(w.dims, R, 7)]
            rows = h.info.nsegs if a.op == "ttm" else w.dims[n]
            width = R * R if a.op == "ttmc" else R  # SpTTMc: R per mode, Kronecker width R^2
            out = torch.empty((rows, width), device="cuda")

            def call():
                if a.op == "ttm":
                    P.fcoo_ttm(h, fs[n], R, out)
                elif a.op == "ttmc":
                    P.fcoo_ttmc(h, fs, out)
                else:
                    P.fcoo_mttkrp(h, fs, R, out)

            for _ in range(3):
                call()
            extra = {}
            if a.flush:
                scratch = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
                times = []
                for _ in range(a.reps):
                    scratch.fill_(1.0)  # evicts the previous rep's factors and stream from L2
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    call()
                    e1.record()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1))
                times.sort()
                ms = times[len(times) // 2]
                extra = {"protocol": "cold L2 (2x L2 scratch write before each rep), per-rep events",
                         "ms_min": round(times[0], 4), "ms_median": round(ms, 4)}
                del scratch
            else:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(a.reps):
                    call()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.reps
            if a.op == "ttm":  # stream (index + value + bf + sf) + U + semi-sparse output
                ntl = h.info.ntiles
                b = nnz * 8 + (nnz + 7) // 8 + 4 * ((ntl + 31) // 32) + 4 * w.dims[n] * R + 4 * h.info.nsegs * R
            elif a.op == "ttmc":  # stream + the two factors + the I_n x R^2 output
                b = compulsory_bytes(w.dims, nnz, n, R, h.info.tile_nnz) - 4 * w.dims[n] * R + 4 * w.dims[n] * width
            else:
                b = compulsory_bytes(w.dims, nnz, n, R, h.info.tile_nnz)
            flops = {"ttm": 2 * R, "ttmc": 2 * width + 1}.get(a.op, N * R) * nnz
            print(json.dumps({"layout": a.layout, "workload": a.workload,
                              "op": a.op, "desc": a.desc, "mode": n, "R": R, "tile": h.info.tile_nnz, "build_ms": round(build_ms, 2), "ms": round(ms, 4),
                              "gnnz_s": round(nnz / ms / 1e6, 2), "gflops": round(flops / ms / 1e6, 1),
                              "hbm_frac": round(b / (ms / 1e3) / 1e9 / peak, 4), **extra}),
                  flush=True)
        h.destroy()


if __name__ == "__main__":
    main()
