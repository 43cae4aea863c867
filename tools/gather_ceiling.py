"""Run the X1 gather-ceiling microbenchmark on cuda:0 and print JSON lines.

python tools/gather_ceiling.py  ->  rows/s and GB/s of random R-wide fp32 row gathers for table
sizes from L1-resident to beyond L2, uniform and Zipf(0.5) index laws.
"""
import ctypes
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libgather.so")


def build():
    src = os.path.join(HERE, "gather_ceiling.cu")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-o", LIB, src])
    return LIB


def main():
    import numpy as np
    import torch

    import gen
    L = ctypes.CDLL(build())
    L.gather_bench.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    n = 64 * 1024 * 1024
    out = torch.zeros(1 << 20, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for R in (16, 32, 64):
        for rows in (256, 1024, 4096, 16384, 65536, 262144, 1048576, 4194304):
            if rows * R * 4 > 2 << 30:
                continue
            table = torch.rand(rows, R, device="cuda")
            for law, alpha in (("uniform", 0.0), ("zipf0.5", 0.5)):
                if law == "uniform":
                    idx = torch.randint(0, rows, (n,), device="cuda", dtype=torch.int32)
                else:
                    # Zipf(alpha) ranks by inverse CDF on the device, then a random relabelling
                    p = torch.arange(1, rows + 1, dtype=torch.float64, device="cuda") ** -alpha
                    c = torch.cumsum(p, 0) / p.sum()
                    u = torch.rand(n, dtype=torch.float64, device="cuda")
                    r = torch.clamp(torch.searchsorted(c, u), max=rows - 1)
                    perm = torch.randperm(rows, device="cuda")
                    idx = perm[r].to(torch.int32).contiguous()
                ms = ctypes.c_float(0)
                rc = L.gather_bench(table.data_ptr(), idx.data_ptr(), n, R, out.data_ptr(), s, 5, ctypes.byref(ms))
                t = ms.value / 1e3
                print(json.dumps({"R": R, "rows": rows, "table_MB": rows * R * 4 / 1e6, "law": law,
                                  "grows_per_s": n / t / 1e9, "gather_TBps": n * R * 4 / t / 1e12, "rc": rc}),
                      flush=True)
                del idx


if __name__ == "__main__":
    main()
