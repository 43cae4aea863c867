"""One fcoo_ttm launch per brainq mode (R=16, automatic tile), for ncu: python tools/prof_ttm.py [--blocked]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import gen
    import paper_1705_09905_b200 as P
    w, idx, val = gen.workload("brainq")
    coo = P.Coo.from_numpy(w.dims, idx, val)
    R = 16
    blocked = "--blocked" in sys.argv
    for n in range(3):
        h = P.fcoo_build(coo, n, op=P.OP_TTM, blocked=blocked)
        U = torch.from_numpy(gen.uniform((w.dims[n], R), 61, n)).cuda()
        out = torch.empty((h.info.nfib, R), device="cuda")
        P.fcoo_ttm(h, U, R, out)
        torch.cuda.synchronize()
        h.destroy()


if __name__ == "__main__":
    main()
