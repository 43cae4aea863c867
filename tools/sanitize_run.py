"""Small end-to-end run that reaches every engine specialisation used at scale (staged float4 path at
R=16/32/64, scalar path, TTM, fp64 CP fit mode, sharded handles, deterministic handles, the blocked
SpMTTKRP / SpTTM, the row-partitioned distributed path) — the workload for
compute-sanitizer memcheck / racecheck / synccheck.

compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import gen
    import paper_1705_09905_b200 as P
    dims = (300, 200, 250)
    idx, val = gen.coo(dims, 30000, (0.8, 0.5, 0.5), 3)
    coo = P.Coo.from_numpy(dims, idx, val)
    for R in (16, 32, 64, 5):
        fs = [torch.from_numpy(f).cuda() for f in gen.factors(dims, R, 4)]
        for n in range(3):
            h = P.fcoo_build(coo, n, tile_nnz=128)
            out = torch.empty((dims[n], R), device="cuda")
            P.fcoo_mttkrp(h, fs, R, out)
            P.fcoo_set_shard(h, 1, 3)
            P.fcoo_mttkrp(h, fs, R, out)
            h.destroy()
            t = P.fcoo_build(coo, n, op=P.OP_TTM, tile_nnz=64)
            yo = torch.empty((t.info.nsegs, R), device="cuda")
            P.fcoo_ttm(t, fs[n], R, yo)
            t.destroy()
    # SpTTMc: staged register-tiled kernels (4x8, 2x4, 1x2, scalar-copy variant) and the unstaged one
    for ranks in ((32, 32), (16, 16), (8, 8), (2, 16), (3, 5)):
        for n in range(3):
            rk = [1, 1, 1]
            others = [m for m in range(3) if m != n]
            rk[others[0]], rk[others[1]] = ranks
            fs = [torch.from_numpy(gen.uniform((d, r), 6, m)).cuda() for m, (d, r) in enumerate(zip(dims, rk))]
            h = P.fcoo_build(coo, n, tile_nnz=64)
            out = torch.empty((dims[n], ranks[0] * ranks[1]), device="cuda")
            P.fcoo_ttmc(h, fs, out)
            h.destroy()
    # 128-bit build keys (65 key bits)
    wd = ((1 << 32) - 1, (1 << 32) - 1, 2)
    widx = np.stack([(np.arange(2000, dtype=np.uint64) * np.uint64(2654435761 + 2 * m) % np.uint64(wd[m]))
                     .astype(np.uint32) for m in range(3)])
    wc = P.Coo.from_numpy(wd, widx, np.ones(2000, np.float32))
    for n in range(3):
        P.fcoo_build(wc, n, tile_nnz=64, keep_perm=True).destroy()
    # CP-ALS: eager first iteration, the captured graph for the rest, the exact-fit recompute
    fs = [torch.from_numpy(f).cuda() for f in gen.factors(dims, 8, 5)]
    P.cp_als(coo, 8, 4, fs, tile_nnz=64)
    # deterministic handles: tile partials + k_combine_boundaries (staged, unstaged, shards, SpTTM,
    # CP-ALS with its fp64 pass), and the library-seeded CP init
    for R in (32, 8):
        fsr = [torch.from_numpy(f).cuda() for f in gen.factors(dims, R, 4)]
        for n in range(3):
            h = P.fcoo_build(coo, n, tile_nnz=64, deterministic=True)
            out = torch.empty((dims[n], R), device="cuda")
            P.fcoo_mttkrp(h, fsr, R, out)
            P.fcoo_set_shard(h, 1, 3)
            P.fcoo_mttkrp(h, fsr, R, out)
            h.destroy()
        t = P.fcoo_build(coo, 1, op=P.OP_TTM, tile_nnz=64, deterministic=True)
        yo = torch.empty((t.info.nsegs, R), device="cuda")
        P.fcoo_ttm(t, fsr[1], R, yo)
        t.destroy()
    fs = [torch.empty((d, 8), device="cuda") for d in dims]
    P.cp_als(coo, 8, 4, fs, tile_nnz=64, seed=3, deterministic=True)
    # blocked layout (round 2): SpMTTKRP float4 shapes with the outer block in shared memory (256 and
    # 512 threads), scalar lanes with global outer rows, shards; the blocked SpTTM (U's block in
    # shared memory, block copies at R = 8 / 16, 3 CTAs per SM) and its fibre map
    for R in (8, 16, 32, 64, 128, 5):
        fsr = [torch.from_numpy(f).cuda() for f in gen.factors(dims, R, 4)]
        for n in range(3):
            for br in (32, 128):
                h = P.fcoo_build(coo, n, tile_nnz=64, blocked=True, block_rows=br)
                out = torch.empty((dims[n], R), device="cuda")
                P.fcoo_mttkrp(h, fsr, R, out)
                P.fcoo_set_shard(h, 1, 3)
                P.fcoo_mttkrp(h, fsr, R, out)
                h.destroy()
                t = P.fcoo_build(coo, n, op=P.OP_TTM, tile_nnz=64, blocked=True, block_rows=br)
                yo = torch.empty((t.info.nfib, R), device="cuda")
                P.fcoo_ttm(t, fsr[n], R, yo)
                t.destroy()
    # row-partitioned path: histogram, bucketing, fake row shards, a 1-rank NCCL distributed build
    # (own-bucket copy), an empty local chunk
    fsr = [torch.from_numpy(f).cuda() for f in gen.factors(dims, 32, 4)]
    for n in range(3):
        hist = P.fcoo_slice_histogram(coo, n).cpu().numpy().view(np.uint32)
        bounds = P.fcoo_row_partition(hist, 3)
        bc, counts = P.fcoo_bucket_rows(coo, n, bounds)
        off = 0
        for k in range(3):
            if counts[k] == 0:
                continue
            part = P.Coo(dims, bc.idx[:, off:off + counts[k]].contiguous(), bc.val[off:off + counts[k]].contiguous())
            off += int(counts[k])
            h = P.fcoo_build(part, n, tile_nnz=64, blocked=True, block_rows=64)
            P.fcoo_set_row_shard(h, k, bounds)
            out = torch.empty((dims[n], 32), device="cuda")
            P.fcoo_mttkrp(h, fsr, 32, out)
            h.destroy()
    comm = P.fcoo_comm_init(0, 1, P.fcoo_comm_unique_id())
    for n in range(3):
        h = P.fcoo_build_distributed(coo, n, comm, tile_nnz=64, blocked=True, block_rows=64)
        out = torch.empty((dims[n], 32), device="cuda")
        P.fcoo_mttkrp(h, fsr, 32, out)
        h.destroy()
    empty = P.Coo(dims, torch.zeros((3, 0), dtype=torch.int32, device="cuda"), torch.zeros(0, device="cuda"))
    h = P.fcoo_build_distributed(empty, 0, comm)
    out = torch.empty((dims[0], 32), device="cuda")
    P.fcoo_mttkrp(h, fsr, 32, out)
    h.destroy()
    comm.destroy()
    # CP-ALS on blocked handles (the default layout)
    fs = [torch.from_numpy(f).cuda() for f in gen.factors(dims, 16, 5)]
    P.cp_als(coo, 16, 4, fs, tile_nnz=64)
    torch.cuda.synchronize()
    print("sanitize_run OK")


if __name__ == "__main__":
    main()
