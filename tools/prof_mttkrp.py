"""Short, profiler-friendly run of the bench workload: build once, then `reps` fcoo_mttkrp calls per
mode.  Used under ncu (launch lists / --set full).  Not a bench number.

python tools/prof_mttkrp.py [--workload nell2] [--R 32] [--reps 3] [--modes 0,1,2] [--tile 256] [--layout blocked|fcoo]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="nell2")
    ap.add_argument("--R", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default=None)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--op", default="mttkrp")
    ap.add_argument("--layout", default="blocked", choices=["blocked", "fcoo"])
    a = ap.parse_args()
    import torch

    import gen
    import paper_1705_09905_b200 as P
    w, idx, val = gen.workload(a.workload)
    coo = P.Coo.from_numpy(w.dims, idx, val)
    modes = [int(m) for m in a.modes.split(",")] if a.modes else list(range(len(w.dims)))
    fs = [torch.from_numpy(f).cuda() for f in gen.factors(w.dims, a.R, 7)]
    for n in modes:
        if a.op == "ttm":
            h = P.fcoo_build(coo, n, op=P.OP_TTM, tile_nnz=a.tile)
            out = torch.empty((h.info.nsegs, a.R), device="cuda")
            for _ in range(a.reps):
                P.fcoo_ttm(h, fs[n], a.R, out)
        elif a.op == "ttmc":
            h = P.fcoo_build(coo, n, tile_nnz=a.tile)
            out = torch.empty((w.dims[n], a.R * a.R), device="cuda")
            for _ in range(a.reps):
                P.fcoo_ttmc(h, fs, out)
        else:
            h = P.fcoo_build(coo, n, tile_nnz=a.tile, blocked=(a.layout == "blocked"))
            out = torch.empty((w.dims[n], a.R), device="cuda")
            for _ in range(a.reps):
                P.fcoo_mttkrp(h, fs, a.R, out)
        torch.cuda.synchronize()
        h.destroy()


if __name__ == "__main__":
    main()
