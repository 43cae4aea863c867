#!/usr/bin/env python
"""bench.py — SpMTTKRP on the F-COO path (arXiv 1705.09905) on B200, one JSON line on rank 0.

Step = one pass of the hot path over one batch of synthetic input: SpMTTKRP on every mode of the
nell-2-shaped tensor (BASELINE.json configs[1]) at R=32, with the F-COO handles (one per mode)
built once and resident in HBM.  value = whole-job GFLOP/s (N*R flops per nonzero per mode,
reading Q18).  Extra keys: roofline (dominant kernel = the MTTKRP segmented reduction, bound =
HBM on the compulsory bytes of SURVEY §8(d)), cpu_baseline (the fp64 oracle on host cores),
e2e (host COO -> device build -> MTTKRP -> host result through the public API), per_mode
(R = 16/32/64 x every mode), clocks, gpu_launches.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
For N > 1 launch with torchrun (one rank per GPU); nonzeros are sharded tile-aligned, factors
replicated, partial outputs combined by an NCCL all-reduce per mode (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "SpMTTKRP GFLOP/s and % HBM roofline per mode at R=16/32/64, 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fcoo", choices=["fcoo", "reference"])
    ap.add_argument("--workload", default="nell2")
    ap.add_argument("--R", type=int, default=32)
    ap.add_argument("--tile", type=int, default=0, help="tile_nnz; 0 = the library's automatic choice")
    ap.add_argument("--layout", default="blocked", choices=["blocked", "fcoo"],
                    help="blocked: FCOO_BUILD_BLOCKED (outer factor block in shared memory, DESIGN.md §5); "
                         "fcoo: the plain F-COO of the paper")
    ap.add_argument("--block-rows", type=int, default=0, help="block_rows for --layout blocked (0 = default)")
    ap.add_argument("--nnz", type=int, default=None, help="override nnz (debug only; not a bench number)")
    ap.add_argument("--combine", default="rows", choices=["rows", "allreduce"],
                    help="N > 1: rows = distributed build (each rank holds the nnz-balanced rows of its chunk "
                         "exchange, owned-rows all-gather); allreduce = redundant build, tile shards, sum all-reduce")
    ap.add_argument("--dist-1rank", action="store_true",
                    help="debug: run the N > 1 row-partitioned code path on one GPU with a 1-rank NCCL comm")
    ap.add_argument("--fused-combine", action="store_true",
                    help="N > 1: combine the ranks' partial outputs in the MTTKRP epilogue through an NVLS "
                         "multicast buffer (fcoo_mttkrp_mc) instead of a separate NCCL all-reduce")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    return ap.parse_args()


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def compulsory_bytes(dims, nnz, mode, R, T):
    """F-COO stream (Table II) + each factor read once + output written once."""
    N = len(dims)
    ntiles = (nnz + T - 1) // T
    b = nnz * (4 * (N - 1) + 4) + (nnz + 7) // 8 + 4 * ((ntiles + 31) // 32)
    b += sum(4 * dims[m] * R for m in range(N) if m != mode) + 4 * dims[mode] * R
    return b


class ClockSampler:
    """NVML SM clock + throttle reasons sampled every 20 ms during the timed region."""
    BAD = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}

    def __init__(self, index):
        self.index, self.samples, self.reasons, self.stop_ev = index, [], set(), threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                 "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                 "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                 "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.th.join()

    def summary(self):
        import statistics
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}

    def rejected(self):
        return bool(self.reasons & self.BAD)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_oracle_baseline(dims, idx, val, R, budget_s=12.0):
    """The oracle as it stands (oracle.mttkrp, fp64, OpenMP over os.cpu_count() threads) on a
    bounded prefix sample of the same workload, every mode.  Returns a cpu_baseline dict."""
    import numpy as np

    import gen
    import oracle
    cores = os.cpu_count() or 1
    fs = gen.factors(dims, R, 7)
    nnz = val.shape[0]
    s = min(nnz, 1_000_000)
    t0 = time.perf_counter()
    oracle.mttkrp(dims, idx[:, :s].copy(), val[:s].copy(), 0, fs, with_D=False, nthreads=cores)
    t1 = time.perf_counter() - t0
    s = int(min(nnz, max(s, s * budget_s / max(t1, 1e-3) / len(dims))))
    si, sv = np.ascontiguousarray(idx[:, :s]), np.ascontiguousarray(val[:s])
    t = 0.0
    for mode in range(len(dims)):
        t0 = time.perf_counter()
        oracle.mttkrp(dims, si, sv, mode, fs, with_D=False, nthreads=cores)
        t += time.perf_counter() - t0
    flops = len(dims) * R * s * len(dims)
    return {"value": flops / t / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"first {s} of {nnz} nonzeros (draw order), SpMTTKRP every mode, R={R}, fp64, "
                      f"{cores} OpenMP threads, {t:.2f} s"}


def run_reference(a):
    """--impl reference: the fp64 oracle on the host cores (this tier's reference arm)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import gen
    import oracle
    w = gen.WORKLOADS[a.workload]
    nnz = a.nnz or w.nnz
    idx, val = gen.coo(w.dims, nnz, w.alpha, w.seed)
    R = a.R
    fs = gen.factors(w.dims, R, 7)
    cores = os.cpu_count() or 1
    N = len(w.dims)
    # per-step sample sized so warmup + steps fit in ~3 minutes
    s = min(nnz, 500_000)
    t0 = time.perf_counter()
    oracle.mttkrp(w.dims, idx[:, :s].copy(), val[:s].copy(), 0, fs, with_D=False, nthreads=cores)
    t1 = max(time.perf_counter() - t0, 1e-4)
    per_step = 150.0 / max(1, a.steps + a.warmup)
    s = int(min(nnz, max(10_000, s * per_step / t1 / N)))
    si, sv = np.ascontiguousarray(idx[:, :s]), np.ascontiguousarray(val[:s])

    def step():
        for mode in range(N):
            oracle.mttkrp(w.dims, si, sv, mode, fs, with_D=False, nthreads=cores)

    for _ in range(a.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()
    el = time.perf_counter() - t0
    flops = N * R * s * N * a.steps
    v = flops / el / 1e9
    sample = (f"first {s} of {nnz} nonzeros (draw order) per step, SpMTTKRP every mode, R={R}, fp64, "
              f"{cores} OpenMP threads")
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": el / a.steps * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{w.name}-shaped {'x'.join(map(str, w.dims))}, {nnz} nnz, alpha {list(w.alpha)}",
                   "R": R, "modes": list(range(N))},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": sample},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import numpy as np
    import torch
    import torch.distributed as dist

    import gen
    import paper_1705_09905_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    w = gen.WORKLOADS[a.workload]
    nnz = a.nnz or w.nnz
    dims = list(w.dims)
    N = len(dims)
    R, T = a.R, a.tile
    idx_np, val_np = gen.coo(dims, nnz, w.alpha, w.seed)
    coo = P.Coo.from_numpy(dims, idx_np, val_np)
    torch.cuda.synchronize()

    comm = P.comm_from_process_group() if world > 1 else None
    if a.dist_1rank and world == 1:
        comm = P.fcoo_comm_init(0, 1, P.fcoo_comm_unique_id())
    blocked = a.layout == "blocked"
    bkw = dict(blocked=blocked, block_rows=a.block_rows) if blocked else {}
    P.fcoo_build(coo, 0, tile_nnz=T, **bkw).destroy()  # warm-up: module load, allocator, CUB tuning
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    row_part = (world > 1 or a.dist_1rank) and a.combine == "rows" and not a.fused_combine
    # this rank's chunk of the input (draw order): the distributed build starts from it
    lo_q, hi_q = nnz * rank // world, nnz * (rank + 1) // world
    chunk = P.Coo(dims, coo.idx[:, lo_q:hi_q].contiguous(), coo.val[lo_q:hi_q].contiguous()) if row_part else None

    def build_all(c, ch, s=None):
        # N > 1, rows: fcoo_build_distributed = histogram, all-reduce, nnz-balanced row ranges, bucket
        # exchange, build of this rank's rows (SURVEY §8(e) owned-rows alternative, §8(f)-4);
        # allreduce: fcoo_build_sharded = the redundant build + this rank's tile-aligned slice (§8(e) v1)
        if row_part:
            return [P.fcoo_build_distributed(ch, n, comm, tile_nnz=T, stream=s, **bkw) for n in range(N)]
        if world > 1:
            return [P.fcoo_build_sharded(c, n, comm, tile_nnz=T, stream=s, **bkw) for n in range(N)]
        return [P.fcoo_build(c, n, tile_nnz=T, stream=s, **bkw) for n in range(N)]

    H = build_all(coo, chunk)
    T = H[0].info.tile_nnz  # the tile actually used (0 = automatic)
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t0) * 1e3

    def factors(R_):
        return [torch.from_numpy(f).to(dev) for f in gen.factors(dims, R_, 7)]

    fs = factors(R)
    outs = [torch.empty((dims[n], R), device=dev) for n in range(N)]
    flops_step = N * R * nnz * N  # every mode
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(N)]

    mc = None
    if a.fused_combine and world > 1:  # one multicast-bound output buffer, reused by every mode
        mc = P.McBuffer(comm, max(dims) * R)

    def step(record=None):
        for n in range(N):
            if record is not None:
                record[n][0].record(stream)
            if mc is not None:
                P.fcoo_mttkrp_mc(H[n], fs, R, mc, stream)
            else:
                P.fcoo_mttkrp(H[n], fs, R, outs[n], stream)
            if record is not None:
                record[n][1].record(stream)

    def timed(K):
        """K steps bracketed by barrier + synchronize; per-mode launch durations on the stream."""
        per_mode = np.zeros(N)
        starts, ends = [], []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = P.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(N)] for _ in range(K)]
        e0.record(stream)
        for k in range(K):
            step(evs[k])
        e1.record(stream)
        torch.cuda.synchronize()
        launches = P.launch_count() - l0
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        for k in range(K):
            for n in range(N):
                per_mode[n] += evs[k][n][0].elapsed_time(evs[k][n][1])
        per_mode /= K
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            pm = torch.tensor(per_mode, device=dev, dtype=torch.float64)
            dist.all_reduce(pm, op=dist.ReduceOp.MAX)
            per_mode = pm.cpu().numpy()
        return ms, per_mode, launches

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    with clk:
        ms, per_mode_ms, launches = timed(a.steps)
    if clk.rejected():  # throttled: re-measure once
        clk = ClockSampler(local)
        with clk:
            ms, per_mode_ms, launches = timed(a.steps)

    value = flops_step * a.steps / (ms / 1e3) / 1e9
    peak, peak_src = hbm_peak()
    bytes_modes = [compulsory_bytes(dims, nnz, n, R, T) for n in range(N)]
    # dominant kernel: the MTTKRP segmented reduction; per-launch algorithmic bytes / launch time.
    # N > 1: the N ranks move the whole job's bytes in the max-rank time, against N GPUs' HBM
    achieved = sum(bytes_modes) / (sum(per_mode_ms) / 1e3) / 1e9
    peak_job = peak * world
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            key = f"{a.workload}/R{R}/T{T}" + ("/blocked" if blocked else "")
            if key in tj:
                traffic = tj[key]
        except Exception:
            pass
    kname = "k_mttkrp_blocked (fcoo_mttkrp, blocked layout)" if blocked else "k_segreduce_staged (fcoo_mttkrp)"
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak_job, "unit": "GB/s", "frac": achieved / peak_job,
                "traffic": traffic, "peak_source": peak_src + (f" x {world} GPUs" if world > 1 else ""),
                "kernel": kname, "bytes_per_launch": {f"mode{n}": int(b) for n, b in enumerate(bytes_modes)},
                "bytes_definition": "SURVEY §8(d): Table II F-COO stream + each factor once + output once"}
    if world > 1:
        roofline["per_rank_frac"] = achieved / world / peak
    if blocked:  # what the blocked stream actually holds (packed words + values + bf + sf)
        roofline["stream_bytes_per_launch"] = {f"mode{n}": int(H[n].info.nstream * (4 * H[n].info.n_words + 4)
                                                                + H[n].info.nstream // 8) for n in range(N)}
    # the binding on-chip ceiling: the L1TEX data pipe that row gathers go through,
    # measured as a hardware property by tools/gather_ceiling.py (profiles/round2/gather_ceiling_
    # shapes.jsonl): random R-wide rows, float4 lanes, L2-resident table; the blocked kernel reads
    # one row per nonzero from shared memory and N-2 from L2 (path LDG+LDS), the plain F-COO
    # kernel N-1 from L2 (path LDG)
    gceil = None
    try:
        rows = [json.loads(l) for l in open(os.path.join(ROOT, "profiles", "round2", "gather_ceiling_shapes.jsonl"))
                if l.startswith("{")]
        want = "LDG+LDS" if blocked and N == 3 else "LDG"
        cands = [r["grows_per_s"] for r in rows if r["R"] == R and r["path"] == want and r["rows"] >= 9184
                 and r["active_groups"] == 1.0 and r["lanes_per_row"] == R // 4]
        gceil = max(cands) if cands else None
    except Exception:
        pass
    rows_per_s = nnz * (N - 1) * N / (sum(per_mode_ms) / 1e3) / 1e9
    result_gather = {"bound": "l1tex_gather", "achieved": rows_per_s, "peak": gceil, "unit": "G rows/s",
                     "frac": (rows_per_s / gceil) if gceil else None,
                     "note": "(N-1) factor rows per nonzero; peak = random-row rate of the same access mix "
                             "measured by tools/gather_ceiling.py at this R (L2-resident table)"}

    result = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{w.name}-shaped {'x'.join(map(str, dims))}, {nnz} nnz, Zipf alpha {list(w.alpha)}, "
                               f"seed {w.seed}",
                   "R": R, "modes": list(range(N)), "tile_nnz": T, "layout": a.layout,
                   "block_rows": H[0].info.block_rows if blocked else None,
                   "parallelism": (f"row-partitioned x{world} (distributed build, nnz-balanced index-mode row "
                                   "ranges per mode), factors replicated, owned-rows all-gather per mode" if row_part else
                                   f"nnz-sharded x{world}, factors replicated, "
                                   + ("combine fused into the MTTKRP epilogue (NVLS multicast)" if mc is not None
                                      else "NCCL all-reduce per mode")) if world > 1
                   else "1 GPU",
                   "l2": "inputs larger than L2: F-COO stream %.2f GB per mode vs 126 MB L2; no explicit flush"
                         % (bytes_modes[0] / 1e9)},
        "nnz_per_s": nnz * N * a.steps / (ms / 1e3),
        "per_mode_ms": [float(x) for x in per_mode_ms],
        "per_mode_hbm_frac": [float(b / (t / 1e3) / 1e9 / peak_job) for b, t in zip(bytes_modes, per_mode_ms)],
        "roofline": roofline, "roofline_gather": result_gather, "gpu_launches": int(launches),
        "clocks": clk.summary(), "build_ms_all_modes": build_ms,
    }

    # ---- per-mode x R sweep (metric: per mode at R=16/32/64) ----
    if not a.no_sweep:
        sweep = []
        for Rs in (16, 32, 64):
            fsr = factors(Rs)
            for n in range(N):
                o = torch.empty((dims[n], Rs), device=dev)
                for _ in range(2):
                    P.fcoo_mttkrp(H[n], fsr, Rs, o, stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 10
                torch.cuda.synchronize()
                e0.record(stream)
                for _ in range(reps):
                    P.fcoo_mttkrp(H[n], fsr, Rs, o, stream)
                e1.record(stream)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / reps
                if world > 1:
                    tt = torch.tensor([t], device=dev, dtype=torch.float64)
                    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                    t = float(tt.item())
                b = compulsory_bytes(dims, nnz, n, Rs, T)
                sweep.append({"R": Rs, "mode": n, "ms": t, "gflops": N * Rs * nnz / (t / 1e3) / 1e9,
                              "hbm_frac": b / (t / 1e3) / 1e9 / peak_job})
        result["per_mode"] = sweep

    def timed_host(step, steps):
        step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / steps
        if world > 1:
            tt = torch.tensor([t], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    # ---- e2e: the public call with HOST buffers.  The F-COO is built and resident once (the
    # paper transfers it once); every step uploads the factors from pinned host memory,
    # runs fcoo_mttkrp on every mode and reads every output back to the host. ----
    if not a.no_e2e:
        f_h = [f.cpu().pin_memory() for f in fs]
        o_h = [torch.empty((dims[n], R)).pin_memory() for n in range(N)]
        fd = [torch.empty_like(f, device=dev) for f in f_h]
        # copies run on their own stream and overlap the MTTKRPs: the factors mode 0 needs go up
        # first, mode 0 starts as soon as they land; each output goes down while the next mode runs
        cs = torch.cuda.Stream(device=dev)
        # mode order that exposes the least copy time: first the mode whose input factors are
        # smallest (the upload it waits for), last the mode with the smallest output (the download
        # left after the last kernel); the step still runs every mode once
        fbytes = [dims[m] * R * 4 for m in range(N)]
        first = min(range(N), key=lambda n: sum(fbytes) - fbytes[n])
        rest = sorted((m for m in range(N) if m != first), key=lambda m: -fbytes[m])
        mode_order = [first] + rest
        up_order = [m for m in range(N) if m != first] + [first]
        up_ev = [torch.cuda.Event() for _ in range(N)]
        out_ev = [torch.cuda.Event() for _ in range(N)]

        def e2e_call_step():
            with torch.cuda.stream(cs):
                for m in up_order:
                    fd[m].copy_(f_h[m], non_blocking=True)
                    up_ev[m].record(cs)
            for n in mode_order:
                for m in range(N):
                    if m != n:
                        stream.wait_event(up_ev[m])
                P.fcoo_mttkrp(H[n], fd, R, outs[n], stream)
                out_ev[n].record(stream)
                cs.wait_event(out_ev[n])
                with torch.cuda.stream(cs):
                    o_h[n].copy_(outs[n], non_blocking=True)
            torch.cuda.synchronize()

        t = timed_host(e2e_call_step, max(a.e2e_steps, 10))
        result["e2e"] = {"value": flops_step / (t / 1e3) / 1e9, "unit": "GFLOP/s",
                         "h2d_bytes_per_step": int(sum(f.numel() * 4 for f in f_h)),
                         "d2h_bytes_per_step": int(sum(o.numel() * 4 for o in o_h)), "ms_per_step": t,
                         "what": "pinned host factors -> device, fcoo_mttkrp every mode, outputs -> pinned host "
                                 "(copies on a second stream, overlapping the MTTKRPs; modes ordered "
                                 f"{mode_order} so the exposed upload/download is smallest); "
                                 "F-COO handles resident (built once, P:L369)"}

    # ---- e2e_with_build: host COO (pinned) -> device, build every mode, MTTKRP every mode -> host ----
    if not a.no_e2e:
        # rows: each rank uploads only its own chunk of the COO (the distributed build exchanges the rest)
        qs = slice(lo_q, hi_q) if row_part else slice(0, nnz)
        idx_h = torch.from_numpy(np.ascontiguousarray(idx_np[:, qs]).view(np.int32)).pin_memory()
        val_h = torch.from_numpy(np.ascontiguousarray(val_np[qs])).pin_memory()
        h2d = idx_h.numel() * 4 + val_h.numel() * 4 + sum(f.numel() * 4 for f in f_h)
        d2h = sum(o.numel() * 4 for o in o_h)

        def e2e_step():
            idx_d = idx_h.to(dev, non_blocking=True)
            val_d = val_h.to(dev, non_blocking=True)
            fd = [f.to(dev, non_blocking=True) for f in f_h]
            c = P.Coo(dims, idx_d, val_d)
            hs = build_all(None if row_part else c, c if row_part else None, stream)
            for n in range(N):
                P.fcoo_mttkrp(hs[n], fd, R, outs[n], stream)
                o_h[n].copy_(outs[n], non_blocking=True)
            torch.cuda.synchronize()
            for h in hs:
                h.destroy()

        t = timed_host(e2e_step, a.e2e_steps)
        result["e2e_with_build"] = {"value": flops_step / (t / 1e3) / 1e9, "unit": "GFLOP/s",
                                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": t,
                                    "what": "pinned host COO + factors -> device, fcoo_build every mode, fcoo_mttkrp "
                                            "every mode, outputs -> host"}

    if rank == 0 and world == 1 and not a.no_cpu:
        result["cpu_baseline"] = cpu_oracle_baseline(dims, idx_np, val_np, R)
    if rank == 0:
        print(json.dumps(result))
    for h in H:
        h.destroy()
    if comm is not None:
        comm.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
