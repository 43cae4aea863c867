"""Experiment: does blocking the nonzero order on one product mode give the co-resident tiles of an
SM a shared factor-row window (L1 reuse)?

Emulation without any library change: for mode n and product mode b, relabel the index mode as
i_n' = blk(i_b) * I_n + i_n with blk(i) = i * K // I_b, so the F-COO sort key becomes
(blk, i_n, product modes ...) and every slice splits into <= K segments.  The timed MTTKRP writes
K * I_n rows (the real blocked kernel would red.add them into I_n rows).  Not a bench number.

python tools/block_experiment.py [--workload nell2] [--R 32] [--K 1,8,16,32,64] [--which outer|inner]
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
    ap.add_argument("--R", type=int, default=32)
    ap.add_argument("--K", default="1,4,8,16,32,64,128")
    ap.add_argument("--which", default="outer,inner")
    ap.add_argument("--modes", default=None)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import numpy as np
    import torch

    import gen
    import paper_1705_09905_b200 as P
    w, idx, val = gen.workload(a.workload)
    N = len(w.dims)
    R = a.R
    modes = [int(m) for m in a.modes.split(",")] if a.modes else list(range(N))
    for n in modes:
        prod = sorted([m for m in range(N) if m != n], key=lambda m: (w.dims[m], m))
        for which in a.which.split(","):
            b = prod[0] if which == "outer" else prod[-1]
            for K in [int(k) for k in a.K.split(",")]:
                if K > w.dims[b]:
                    continue
                blk = (idx[b].astype(np.int64) * K) // w.dims[b]
                idx2 = idx.copy()
                idx2[n] = (blk * w.dims[n] + idx[n]).astype(np.uint32)
                dims2 = list(w.dims)
                dims2[n] = K * w.dims[n]
                coo = P.Coo.from_numpy(dims2, idx2, val)
                h = P.fcoo_build(coo, n)
                fs = [torch.from_numpy(f).cuda() for f in gen.factors(dims2, R, 7)]
                out = torch.empty((dims2[n], R), device="cuda")
                for _ in range(2):
                    P.fcoo_mttkrp(h, fs, R, out)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(a.reps):
                    P.fcoo_mttkrp(h, fs, R, out)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.reps
                print(json.dumps({"workload": a.workload, "mode": n, "R": R, "block_mode": b, "which": which,
                                  "K": K, "nsegs": h.info.nsegs, "tile": h.info.tile_nnz, "ms": round(ms, 4),
                                  "gnnz_s": round(val.shape[0] / ms / 1e6, 2)}), flush=True)
                h.destroy()
                del coo, fs, out
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
