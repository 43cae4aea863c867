"""Time fcoo_build_distributed against fcoo_build on one GPU with a 1-rank NCCL comm (the per-rank
work of the distributed build without the network: histogram, bucketing, own-bucket copy, build).

python tools/dist_build_time.py [--workload nell2] [--blocked]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="nell2")
    ap.add_argument("--blocked", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    import gen
    import paper_1705_09905_b200 as P
    w, idx, val = gen.workload(a.workload)
    coo = P.Coo.from_numpy(w.dims, idx, val)
    comm = P.fcoo_comm_init(0, 1, P.fcoo_comm_unique_id())
    kw = dict(blocked=True) if a.blocked else {}

    def timeit(fn):
        fn().destroy()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            fn().destroy()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / a.reps * 1e3

    for n in range(len(w.dims)):
        t_plain = timeit(lambda: P.fcoo_build(coo, n, **kw))
        t_dist = timeit(lambda: P.fcoo_build_distributed(coo, n, comm, **kw))
        def host_ms(fn):
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(a.reps):
                fn()
            torch.cuda.synchronize()
            return (time.perf_counter() - t0) / a.reps * 1e3

        hist = P.fcoo_slice_histogram(coo, n).cpu().numpy().view("uint32")
        t_hist = host_ms(lambda: P.fcoo_slice_histogram(coo, n))
        bounds = P.fcoo_row_partition(hist, 8)
        t_bucket = host_ms(lambda: P.fcoo_bucket_rows(coo, n, bounds))
        b1 = P.fcoo_row_partition(hist, 1)
        bc, _ = P.fcoo_bucket_rows(coo, n, b1)
        t_bucket1 = host_ms(lambda: P.fcoo_bucket_rows(coo, n, b1))
        t_build_b = timeit(lambda: P.fcoo_build(bc, n, **kw))
        h = P.fcoo_build(bc, n, **kw)
        t_rows = host_ms(lambda: P.fcoo_set_row_shard(h, 0, b1))
        h.destroy()
        print(json.dumps({"workload": a.workload, "mode": n, "blocked": a.blocked, "nnz": int(val.shape[0]),
                          "build_ms": round(t_plain, 2), "build_distributed_1rank_ms": round(t_dist, 2),
                          "slice_histogram_ms": round(t_hist, 2), "bucket_rows_1rank_ms": round(t_bucket1, 2),
                          "bucket_rows_8ranks_ms": round(t_bucket, 2), "build_of_bucketed_ms": round(t_build_b, 2),
                          "set_row_shard_ms": round(t_rows, 2)}),
              flush=True)
    comm.destroy()


if __name__ == "__main__":
    main()
