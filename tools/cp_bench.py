"""Time cp_als (the C-ABI CP-ALS) on a workload and report the per-iteration time and the share of
SpMTTKRP in it ("most of execution time ... spent on the SpMTTKRP operation").

python tools/cp_bench.py [--workload order4] [--R 32] [--iters 20]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="order4")
    ap.add_argument("--R", type=int, default=32)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--tile", type=int, default=0)
    a = ap.parse_args()
    import torch

    import gen
    import paper_1705_09905_b200 as P
    w, idx, val = gen.workload(a.workload)
    coo = P.Coo.from_numpy(w.dims, idx, val)
    N = len(w.dims)

    def init():
        return [torch.from_numpy(f).cuda() for f in gen.factors(w.dims, a.R, 9)]

    def run(iters):
        fs_ = init()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lam_, trace_ = P.cp_als(coo, a.R, iters, fs_, tile_nnz=a.tile)
        torch.cuda.synchronize()
        return time.perf_counter() - t0, fs_, trace_

    run(1)  # warm-up (module load, allocator)
    k1 = max(1, a.iters // 4)
    one = min(run(k1)[0] for _ in range(2))
    total, fs, trace = run(a.iters)
    total = min(total, run(a.iters)[0])
    per_iter_s = (total - one) / (a.iters - k1)
    one = one - (k1 - 1) * per_iter_s
    # MTTKRP alone, every mode (same handles layout)
    hs = [P.fcoo_build(coo, n, tile_nnz=a.tile) for n in range(N)]
    outs = [torch.empty((w.dims[n], a.R), device="cuda") for n in range(N)]
    for n in range(N):
        P.fcoo_mttkrp(hs[n], fs, a.R, outs[n])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        for n in range(N):
            P.fcoo_mttkrp(hs[n], fs, a.R, outs[n])
    e1.record()
    torch.cuda.synchronize()
    mttkrp_iter = e0.elapsed_time(e1) / 5 / 1e3
    per_iter = per_iter_s
    print(json.dumps({"workload": a.workload, "dims": list(w.dims), "nnz": int(val.shape[0]), "R": a.R,
                      "iters": a.iters, "total_s": total, "per_iter_ms": per_iter * 1e3,
                      "setup_ms_est": (one - per_iter) * 1e3, "mttkrp_all_modes_ms": mttkrp_iter * 1e3,
                      "mttkrp_share": mttkrp_iter / per_iter, "fit_first": trace[0], "fit_last": trace[-1]}))


if __name__ == "__main__":
    main()
