"""Run the X1 gather-ceiling microbenchmark (tools/gather_ceiling.cu) on cuda:0; one JSON line per cell.

The on-chip roofline of the SpMTTKRP factor-row gathers as a hardware property (VERDICT r1 item
1a): rows/clk/SM for random R-wide fp32 row gathers, per access shape (float4 / float2 / float
lanes), per data path (LDG, texture, shared memory, and their mixes), per table size (L1/smem-
resident, L2-resident, HBM) and per fraction of active lane-groups.

  python tools/gather_ceiling.py [--quick]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libgather.so")
PATHS = {0: "LDG", 1: "TEX", 2: "LDS", 3: "LDG+TEX", 4: "LDG+LDS", 5: "LDS+TEX", 6: "LDG+LDS+TEX"}


def build():
    src = os.path.join(HERE, "gather_ceiling.cu")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-o", LIB, src])
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--share", action="store_true", help="only the shared-row (warp-cooperative reuse) sweep")
    ap.add_argument("--clock-mhz", type=float, default=1965.0)
    a = ap.parse_args()
    import torch
    L = ctypes.CDLL(build())
    L.gather_bench3.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                                ctypes.POINTER(ctypes.c_double)]
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    out = torch.zeros(1 << 22, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def cell(R, rows, vec, path, act4=4, srows=0, bps=4, steps=400, share=1):
        table = torch.rand(rows, R, device="cuda")
        ms, nr = ctypes.c_float(0), ctypes.c_double(0)
        rc = L.gather_bench3(table.data_ptr(), rows, R, vec, path, srows, act4, share, bps, steps, out.data_ptr(), s, 5,
                             ctypes.byref(ms), ctypes.byref(nr))
        t = ms.value / 1e3
        rps = nr.value / t
        line = {"R": R, "rows": rows, "table_MB": rows * R * 4 / 1e6, "lanes_per_row": R // vec, "vec": vec,
                "path": PATHS[path], "smem_rows": srows, "active_groups": act4 / 4, "ctas_per_sm": bps,
                "groups_sharing_lds_row": share,
                "grows_per_s": rps / 1e9, "rows_per_clk_sm": rps / (nsm * a.clock_mhz * 1e6),
                "bytes_per_clk_sm": rps * R * 4 / (nsm * a.clock_mhz * 1e6), "rc": rc}
        print(json.dumps(line), flush=True)

    if a.share:  # warp-cooperative reuse: lane-groups of a warp reading one shared-memory row
        for R in (16, 32, 64):
            srows = 12288 // R
            for share in (1, 2, 4, 8):
                if share * R // 4 > 32:
                    continue
                cell(R, srows, 4, 2, srows=srows, share=share)
                cell(R, 28818, 4, 4, srows=srows, share=share)
        return
    Rs = (32,) if a.quick else (16, 32, 64)
    for R in Rs:
        srows = 12288 // R  # 48 KB of shared memory: 4 CTAs/SM
        for rows in ((srows, 9184, 28818) if a.quick else (srows, 9184, 28818, 480189)):
            for vec in (4, 2, 1):
                if R // vec > 32:
                    continue
                cell(R, rows, vec, 0)
        for path in (1, 2, 3, 4, 5, 6):
            for rows in (srows, 28818):
                cell(R, rows, 4, path, srows=srows if path in (2, 4, 5, 6) else 0, bps=4)
        for act4 in (1, 2, 3):
            cell(R, 28818, 4, 0, act4=act4)
            cell(R, srows, 4, 2, act4=act4, srows=srows, bps=4)


if __name__ == "__main__":
    main()
