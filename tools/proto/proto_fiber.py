"""EXPERIMENT ONLY: time the blocked / fibre-factored SpMTTKRP prototypes (proto_fiber.cu) against
the library kernel on the nell-2-shaped tensor.  The blocked, padded stream is built here with
torch on the GPU (tooling, not the product path).  Prints JSON lines.

python tools/proto/proto_fiber.py [--R 32] [--modes 0,1,2] [--BR 768,1536] [--var 1,2,3,4] [--tb 512]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libproto.so")


def build():
    src = os.path.join(HERE, "proto_fiber.cu")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC", "-shared", "-o", LIB, src])
    return LIB


class PB(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("pk", "val", "bf", "ff", "sf", "seg_base", "seg_row", "item_blk",
                                                "item_t0", "item_nt", "blk_end", "Uo", "Ui", "out")] + \
               [("ntiles", ctypes.c_int64), ("T", ctypes.c_int), ("BR", ctypes.c_int), ("Io", ctypes.c_int),
                ("IB", ctypes.c_int)]


class PP(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("po", "pi", "val", "bf", "ff", "sf", "seg_base", "seg_row", "item_blk",
                                                "item_t0", "item_nt", "Uo", "Ui", "out")] + \
               [("ntiles", ctypes.c_int64), ("T", ctypes.c_int), ("R", ctypes.c_int), ("BR", ctypes.c_int),
                ("Io", ctypes.c_int)]


def pack_bits(h):
    """bool tensor (len multiple of 32) -> uint32 words LSB-first (as int32 tensor)."""
    import torch
    w = h.view(-1, 32).to(torch.int64) << torch.arange(32, device=h.device, dtype=torch.int64)
    return w.sum(1).to(torch.int64).bitwise_and(0xffffffff).to(torch.uint32).view(torch.int32)


def build_stream(idx, val, dims, mode, BR, T, GPC, zero_pad=False):
    import torch
    dev = idx.device
    prod = sorted([m for m in range(3) if m != mode], key=lambda m: (dims[m], m))
    o, i = prod
    io, ii, iN = idx[o].long(), idx[i].long(), idx[mode].long()
    nblk = (dims[o] + BR - 1) // BR if BR else 1
    blk = io // BR if BR else torch.zeros_like(io)
    key = ((blk * dims[mode] + iN) * dims[o] + io) * dims[i] + ii
    order = torch.argsort(key)
    blk_s, n_s, o_s, i_s, v_s = blk[order], iN[order], io[order], ii[order], val[order]
    counts = torch.bincount(blk_s, minlength=nblk)
    padded = ((counts + T - 1) // T) * T
    start = torch.cumsum(counts, 0) - counts
    pstart = torch.cumsum(padded, 0) - padded
    total = int(padded.sum())
    nnz = idx.shape[1]
    src = torch.empty(total, dtype=torch.int64, device=dev)
    # default: pad entries copy the block's last nonzero
    blk_of_pos = torch.repeat_interleave(torch.arange(nblk, device=dev), padded)
    last = start + counts - 1
    src[:] = last[blk_of_pos]
    pos = pstart[blk_s] + (torch.arange(nnz, device=dev) - start[blk_s])
    src[pos] = torch.arange(nnz, device=dev)
    isreal = torch.zeros(total, dtype=torch.bool, device=dev)
    isreal[pos] = True
    S_blk, S_n, S_o, S_i = blk_s[src], n_s[src], o_s[src], i_s[src]
    S_v = torch.where(isreal, v_s[src], torch.zeros((), device=dev))
    blk_end = (pstart + counts).to(torch.int64)
    head = torch.ones(total, dtype=torch.bool, device=dev)
    head[1:] = (S_blk[1:] != S_blk[:-1]) | (S_n[1:] != S_n[:-1])
    fh = head.clone()
    fh[1:] |= S_o[1:] != S_o[:-1]
    if zero_pad:
        head &= isreal
        fh &= isreal
    ntiles = total // T
    seg_row = S_n[head].to(torch.int32)
    ch = torch.cumsum(head.to(torch.int64), 0)
    seg_base = torch.zeros(ntiles + 1, dtype=torch.int64, device=dev)
    tp = torch.arange(ntiles, device=dev) * T
    seg_base[:ntiles] = ch[tp] - head[tp].to(torch.int64)
    seg_base[ntiles] = ch[-1]
    sfb = head[tp]
    sfb = torch.cat([sfb, torch.zeros((-ntiles) % 32 + 32, dtype=torch.bool, device=dev)])
    tile_blk = S_blk[tp]
    # work items: per block, chunks of GPC tiles
    items_blk, items_t0, items_nt = [], [], []
    tb = torch.cumsum(padded // T, 0).tolist()
    t_lo = 0
    for b in range(nblk):
        t_hi = tb[b]
        for t0 in range(t_lo, t_hi, GPC):
            items_blk.append(b)
            items_t0.append(t0)
            items_nt.append(min(GPC, t_hi - t0))
        t_lo = t_hi
    i32 = lambda x: torch.tensor(x, dtype=torch.int32, device=dev)
    IB = max(1, int(dims[i] - 1).bit_length())
    loc = (S_o - S_blk * BR) if BR else S_o
    pk = torch.where(isreal, (loc << IB) | S_i, torch.zeros((), dtype=torch.int64, device=dev))
    pk = pk.bitwise_and(0xffffffff).to(torch.uint32).view(torch.int32) if int(loc.max()).bit_length() + IB <= 32 else None
    return dict(pk=pk, IB=IB, blk_end=blk_end, po=S_o.to(torch.int32), pi=S_i.to(torch.int32), val=S_v.contiguous(), bf=pack_bits(head),
                ff=pack_bits(fh), sf=pack_bits(sfb), seg_base=seg_base.to(torch.int32), seg_row=seg_row,
                item_blk=i32(items_blk), item_t0=i32(items_t0), item_nt=i32(items_nt), ntiles=ntiles, total=total,
                nblk=nblk, o=o, i=i, nsegs=int(head.sum()), nfib=int(fh.sum()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", default="32")
    ap.add_argument("--modes", default="0,1,2")
    ap.add_argument("--BR", default="768,1536")
    ap.add_argument("--var", default="1,2,3,4")
    ap.add_argument("--tb", type=int, default=512)
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--nnz", type=int, default=None)
    ap.add_argument("--once", action="store_true", help="one launch per kernel (for ncu)")
    a = ap.parse_args()
    import numpy as np
    import torch

    import gen
    import paper_1705_09905_b200 as F
    L = ctypes.CDLL(build())
    L.proto_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(PP), ctypes.c_int, ctypes.c_void_p]
    L.proto_blk2.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(PB), ctypes.c_int, ctypes.c_void_p]
    L.proto_blk.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(PB), ctypes.c_int, ctypes.c_void_p]
    assert L.proto_blk_sizeof() == ctypes.sizeof(PB)
    assert L.proto_sizeof() == ctypes.sizeof(PP), (L.proto_sizeof(), ctypes.sizeof(PP))
    w = gen.WORKLOADS["nell2"]
    dims = list(w.dims)
    nnz = a.nnz or w.nnz
    idx_np, val_np = gen.coo(dims, nnz, w.alpha, w.seed)
    dev = torch.device("cuda")
    idx = torch.from_numpy(idx_np.astype(np.int64)).to(dev)
    val = torch.from_numpy(val_np).to(dev)
    coo = F.Coo.from_numpy(dims, idx_np, val_np)
    s = torch.cuda.current_stream()

    def timeit(fn, reps):
        if a.once:
            fn()
            torch.cuda.synchronize()
            return 1.0
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    for R in [int(x) for x in a.R.split(",")]:
        fs = [torch.from_numpy(f).to(dev) for f in gen.factors(dims, R, 7)]
        for mode in [int(x) for x in a.modes.split(",")]:
            H = F.fcoo_build(coo, mode, tile_nnz=a.T)
            ref = torch.empty((dims[mode], R), device=dev)
            ms_lib = timeit(lambda: F.fcoo_mttkrp(H, fs, R, ref, s), a.reps)
            H.destroy()
            print(json.dumps({"R": R, "mode": mode, "var": "library", "ms": ms_lib}), flush=True)
            for BR in [int(x) for x in a.BR.split(",")]:
                for var in [int(x) for x in a.var.split(",")]:
                    if var == 1 and BR != int(a.BR.split(",")[0]):
                        continue
                    GPC = a.tb // (R // 4)
                    if var in (5, 6, 7, 8):
                        st = build_stream(idx, val, dims, mode, BR, a.T, GPC, zero_pad=True)
                        out = torch.zeros((dims[mode], R), device=dev)
                        p = PB()
                        for k in ("pk", "val", "bf", "ff", "sf", "seg_base", "seg_row", "item_blk", "item_t0", "item_nt",
                                  "blk_end"):
                            setattr(p, k, st[k].data_ptr())
                        p.Uo, p.Ui, p.out = fs[st["o"]].data_ptr(), fs[st["i"]].data_ptr(), out.data_ptr()
                        p.ntiles, p.T, p.BR, p.Io, p.IB = st["ntiles"], a.T, BR, dims[st["o"]], st["IB"]
                        nitems = len(st["item_blk"])

                        def run():
                            out.zero_()
                            if var == 8:
                                rc = L.proto_blk2(R, a.tb, ctypes.byref(p), nitems, s.cuda_stream)
                            else:
                                rc = L.proto_blk(var - 5, R, a.tb, ctypes.byref(p), nitems, s.cuda_stream)
                            assert rc == 0, rc
                    if var in (5, 6, 7, 8):
                        if not a.once:
                            run()
                        torch.cuda.synchronize()
                        err = ((out - ref).abs().max() / ref.abs().max()).item()
                        print("DEBUG", out.abs().sum().item(), ref.abs().sum().item(), out[0, :4].tolist(), ref[0, :4].tolist(),
                              (out != ref).sum().item(), file=sys.stderr)
                        ms = timeit(run, a.reps)
                        ms_zero = timeit(lambda: out.zero_(), a.reps)
                        print(json.dumps({"R": R, "mode": mode, "var": var, "BR": BR, "tb": a.tb, "ms": ms - ms_zero,
                                          "ms_lib": ms_lib, "speedup": ms_lib / max(ms - ms_zero, 1e-9), "relerr": err,
                                          "nblk": st["nblk"], "pad_frac": st["total"] / nnz - 1, "nsegs": st["nsegs"],
                                          "fib_per_nnz": st["nfib"] / nnz, "items": nitems}), flush=True)
                        del st, out
                        continue
                    if var == 2 or var == 3:
                        smem = BR * R * 4 + GPC * 204 * 4
                        if smem > 227 * 1024:
                            continue
                    st = build_stream(idx, val, dims, mode, 0 if var == 1 else BR, a.T, GPC)
                    out = torch.zeros((dims[mode], R), device=dev)
                    p = PP()
                    for k in ("po", "pi", "val", "bf", "ff", "sf", "seg_base", "seg_row", "item_blk", "item_t0", "item_nt"):
                        setattr(p, k, st[k].data_ptr())
                    p.Uo, p.Ui, p.out = fs[st["o"]].data_ptr(), fs[st["i"]].data_ptr(), out.data_ptr()
                    p.ntiles, p.T, p.R, p.BR, p.Io = st["ntiles"], a.T, R, BR if var != 1 else dims[st["o"]], dims[st["o"]]
                    nitems = len(st["item_blk"]) if var != 1 else (st["ntiles"] + GPC - 1) // GPC

                    def run():
                        out.zero_()
                        rc = L.proto_run(var, a.tb, ctypes.byref(p), nitems, s.cuda_stream)
                        assert rc == 0, rc

                    if not a.once:
                        run()
                    torch.cuda.synchronize()
                    err = ((out - ref).abs().max() / ref.abs().max()).item()
                    ms = timeit(run, a.reps)
                    ms_zero = timeit(lambda: out.zero_(), a.reps)
                    print(json.dumps({"R": R, "mode": mode, "var": var, "BR": BR, "ms": ms - ms_zero, "ms_lib": ms_lib,
                                      "speedup": ms_lib / max(ms - ms_zero, 1e-9), "relerr": err, "nblk": st["nblk"],
                                      "pad_frac": st["total"] / nnz - 1, "nsegs": st["nsegs"],
                                      "fib_per_nnz": st["nfib"] / nnz, "items": nitems}), flush=True)
                    del st, out


if __name__ == "__main__":
    main()
