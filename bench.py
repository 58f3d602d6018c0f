#!/usr/bin/env python
"""Benchmark: BFS GTEPS on R-MAT (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scale 24] [--algo bfs|sssp|pr|cc|tc] [--source 0]

One step = one full ``bfs(A, source)`` through the public API on the R-MAT
graph of the reference generator (io.py:275-295, seed 1, a/b/c/d =
.57/.19/.19/.05, edge factor 16, symmetrised).  The graph is generated on the
GPU and resident in HBM before timing (cli.py:200-214 excludes load time).
TEPS = stored edges / time (cli.py:222).

Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement for every field.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "BFS GTEPS on RMAT scale-24"
# B200 nominal HBM3e bandwidth (SURVEY §8(d) asks for the fraction of it too)
NOMINAL_HBM_GBS = 8000.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--algo", default="bfs", choices=["bfs"])
    ap.add_argument("--source", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-spmv", action="store_true", help="skip the masked SpMV measurement")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config sweep (BASELINE configs C1-C5, GPU vs C oracle)")
    ap.add_argument("--cpu-cap-s", type=float, default=120.0,
                    help="wall-clock cap for CPU timing legs")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# roofline bookkeeping
# ---------------------------------------------------------------------------


def bench_config(args, n, m):
    """The config object, identical in both arms (same workload, same graph)."""
    return {"workload": f"bfs(A, {args.source}) on rmat-s{args.scale}-e16 symmetrised",
            "n": n, "nnz": m,
            "l2": "inputs larger than L2 (CSR %.2f GB vs 126 MB)" % ((m * 4 + (n + 1) * 8) / 1e9)}


def cpu_model():
    """lscpu's model name (the host the CPU baseline ran on)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


def measured_peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def committed_traffic(kernel):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    p = os.path.join(HERE, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    return d.get(kernel)


def push_level_bytes(n, k, flops, k_next):
    """Algorithmic bytes of one push SpMSpV level: frontier ids +
    two int64 offsets per frontier vertex, one int32 column index per edge,
    the visited bitmap probe (n/8) and the next-frontier bitmap (n/8)."""
    return k * (4 + 2 * 8) + flops * 4 + n / 8 + n / 8 + k_next * (4 + 8)


def ctx_ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def masked_spmv(gb, A, ctx, peak, peak_src, reps=10, density=0.5, graph="rmat"):
    """The second half of the BASELINE metric: masked pull SpMV at the bench
    scale through the public API, w<!m> = A (+.*) x (x dense f64, m a seeded
    50 % mask, complemented; forced pull), timed per kernel with events.
    Algorithmic bytes per SURVEY §8(d): n/8 (mask) + min(2R, n+1)*8 (offsets
    of the R allowed rows) + E_read*4 (their column indices; pattern matrix,
    no values) + n*8 (x, once) + n*8 (w).  Checked against torch index_add."""
    import torch
    from paper_1908_01407_b200.containers import MaskMode, Vector
    n = A.nrows
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
    mbits = (torch.rand(n, device="cuda", generator=g) < density).to(torch.int64)
    u = Vector._wrap(n, None, x, 0.0, np.float64)
    mask = Vector._wrap(n, None, mbits, 0, np.int64)
    sr = gb.builtin_semiring("PlusMultiplies")

    def run():
        d = gb.Descriptor(mask_mode=MaskMode.COMPLEMENT, direction=gb.Direction.FORCE_PULL)
        return gb.mxv(sr, A, u, mask=mask, desc=d), d

    run()
    run()
    torch.cuda.synchronize()
    ctx.profiling(True)
    for _ in range(reps):
        w, d = run()
    torch.cuda.synchronize()
    prof = ctx.prof_read()
    ctx.profiling(False)
    t_ms = float(np.median([t for (kind, _a, t) in prof if kind == 8]))
    off = A._csr.offsets
    deg = torch.diff(off)
    allowed = mbits == 0
    R = int(((deg > 0) & allowed).sum())
    e_read = d.counters.matrix_entries_read
    bytes_alg = n / 8 + min(2 * R, n + 1) * 8 + e_read * 4 + n * 8 + n * 8
    # the gather ceiling of this matrix: stream every column index and gather
    # x[col], nothing else (gb_gather_replay_rate) -- the random 8-byte
    # gathers, not HBM bandwidth, bound a pull over a 134 MB x
    import ctypes
    rate = ctypes.c_double(0)
    st, _k = A._csr.csr_struct(np.float64)
    ctx.call("gb_gather_replay_rate", ctypes.byref(st), ctx_ptr(x), ctypes.byref(rate))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    call_ms = e0.elapsed_time(e1) / reps
    rows = torch.repeat_interleave(torch.arange(n, device="cuda"), deg)
    keep = allowed[rows]
    ref = torch.zeros(n, dtype=torch.float64, device="cuda")
    ref.index_add_(0, rows[keep], x[A._csr.indices.long()[keep]])
    rel = float(((w._vals - ref).abs() / ref.abs().clamp_min(1e-300)).max())
    del rows, keep, ref
    achieved = bytes_alg / (t_ms * 1e-3) / 1e9
    # A/B: the same call through the edge-balanced row tiles (the reference's
    # nonzero split) instead of the row bins (its row split)
    from paper_1908_01407_b200 import kernels as _k
    saved = _k._MV_BINS
    _k._MV_BINS = "0"
    try:
        run()
        torch.cuda.synchronize()
        ctx.profiling(True)
        for _ in range(reps):
            run()
        torch.cuda.synchronize()
        tiles_ms = float(np.median([t for (kind, _a, t) in ctx.prof_read() if kind == 8]))
        ctx.profiling(False)
    finally:
        _k._MV_BINS = saved
    return {"workload": f"mxv(PlusMultiplies f64, A={graph}, x dense, mask=~m, m {density:.0%} "
                        "seeded), forced pull",
            "kernel": "mv_pull_binned (row bins, mask tested per row)",
            "traffic": committed_traffic("mv_pull_binned" if graph == "rmat" else "mv_pull_binned_uniform_striped"),
            "ab_ms": {"row_bins (default; Partition.ROW_SPLIT)": round(t_ms, 4),
                      "row_tiles (edge-balanced)": round(tiles_ms, 4)},
            "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "peak_source": peak_src,
            "frac_vs_nominal_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
            "bytes_alg": int(bytes_alg), "launch_ms": round(t_ms, 4),
            "call_ms": round(call_ms, 4),
            "gather_replay": {
                "what": "gb_gather_replay_rate: stream A's column indices and gather x[col] "
                        "for every stored entry in one pass, nothing else (measured in this "
                        "run) -- the rate the random 8 B gathers allow a one-pass pull; a "
                        "column-striped pull (regular graphs) can exceed it",
                "replay_Ggather_s": round(rate.value / 1e9, 1),
                "achieved_Ggather_s": round(e_read / (t_ms * 1e-3) / 1e9, 1),
                "ratio": round(e_read / (t_ms * 1e-3) / rate.value, 4)},
            "allowed_rows": R,
            "entries_read": int(e_read), "multiplies": int(d.counters.semiring_multiplies),
            "max_rel_err_vs_torch": rel, "tolerance": 1e-12, "parity": rel <= 1e-12}


# ---------------------------------------------------------------------------
# every BASELINE.json config: device time, parity against the C oracle on the
# same CSR, and the C port timed on the host (the reported CPU baseline)
# ---------------------------------------------------------------------------


def _dev_ms(fn, reps, warmup=1):
    import torch
    for _ in range(warmup):
        r = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


def _cpu_s(fn):
    t = time.perf_counter()
    r = fn()
    return time.perf_counter() - t, r


def config_sweep(gb, scales=(16, 20, 22, 24, 26)):
    """BASELINE.json configs C1-C5: one JSON object per config."""
    import torch
    from oracle import cgraph
    from paper_1908_01407_b200.io import rmat_matrix
    cgraph.lib()
    out = {"cpu_threads": cgraph.threads(), "cpu_kind": "port (oracle/cgraph.c, OpenMP)"}

    def host(A):
        return A._csr.offsets.cpu().numpy(), A._csr.indices.cpu().numpy()

    def cleanup():
        gb._lib.context().trim()
        torch.cuda.empty_cache()

    # C1: BFS from 0 on s16
    if 16 in scales:
        A = rmat_matrix(16)
        # a 50 us call is host-bound: warm the host path (CPU clocks, caches)
        # for a few hundred calls before timing
        ms, lv = _dev_ms(lambda: gb.bfs(A, 0), 200, warmup=300)
        rp, ci = host(A)
        cs, (want, _tr) = _cpu_s(lambda: cgraph.bfs(rp, ci, 0))
        out["C1_bfs_s16"] = {"gpu_ms": round(ms, 4), "cpu_ms": round(cs * 1e3, 3), "nnz": A.nnz,
                             "gteps": round(A.nnz / ms / 1e6, 2),
                             "parity": bool(np.array_equal(lv.values, want))}
        A = None
        cleanup()
    # C2: SSSP (min-plus) on s20 with the reference integer weights as f64
    if 20 in scales:
        W = rmat_matrix(20, weighted=True)
        ms, dist = _dev_ms(lambda: gb.sssp(W, 0), 10, warmup=2)
        rp, ci = host(W)
        w = W._csr.dense_values().cpu().numpy()
        cs, (want, _tr) = _cpu_s(lambda: cgraph.sssp(rp, ci, w, 0))
        got = dist.values
        fin = np.isfinite(want)
        rel = float(np.max(np.abs(got[fin] - want[fin]) / np.maximum(np.abs(want[fin]), 1e-300)))
        out["C2_sssp_s20"] = {"gpu_ms": round(ms, 3), "cpu_ms": round(cs * 1e3, 1),
                              "max_rel_err": rel, "tolerance": 1e-5,
                              "parity": bool(rel <= 1e-5 and np.array_equal(np.isinf(got), ~fin))}
        W = None
        cleanup()
        # C4: triangle counting (fused degree-ranked count) on s20 (golden 424,532,724)
        A = rmat_matrix(20)
        ms, cnt = _dev_ms(lambda: gb.triangle_count(A), 5, warmup=2)
        rp, ci = host(A)
        cs, want = _cpu_s(lambda: cgraph.tc(rp, ci))
        out["C4_tc_s20"] = {"gpu_ms": round(ms, 3), "cpu_ms": round(cs * 1e3, 1), "triangles": int(cnt),
                            "parity": bool(int(cnt) == want == 424_532_724)}
        A = None
        cleanup()
    # C3: PageRank 20 iterations (plus-times, dense pull) on s22
    if 22 in scales:
        A = rmat_matrix(22)
        ms, pr = _dev_ms(lambda: gb.pagerank(A, eps=1e-300, max_iters=20), 5, warmup=2)
        rp, ci = host(A)
        cs, (want, _e) = _cpu_s(lambda: cgraph.pagerank(rp, ci, eps=1e-300, max_iters=20))
        l1 = float(np.abs(pr.values - want).sum())
        out["C3_pagerank20_s22"] = {"gpu_ms": round(ms, 3), "cpu_ms": round(cs * 1e3, 1),
                                    "l1_vs_oracle": l1, "tolerance": 1e-6, "parity": bool(l1 <= 1e-6)}
        A = None
        cleanup()
    # C5: BFS + connected components on s24 and s26 (one GPU)
    for sc in (24, 26):
        if sc not in scales:
            continue
        try:
            A = rmat_matrix(sc)
            bms, lv = _dev_ms(lambda: gb.bfs(A, 0), 5)
            cms, lab = _dev_ms(lambda: gb.connected_components(A), 2)
            rp, ci = host(A)
            bcs, (want, _tr) = _cpu_s(lambda: cgraph.bfs(rp, ci, 0))
            ccs, (wlab, _t2) = _cpu_s(lambda: cgraph.cc(rp, ci))
            out[f"C5_bfs_cc_s{sc}"] = {
                "n": A.nrows, "nnz": A.nnz, "bfs_gpu_ms": round(bms, 3),
                "bfs_gteps": round(A.nnz / bms / 1e6, 1), "bfs_cpu_ms": round(bcs * 1e3, 1),
                "cc_gpu_ms": round(cms, 3), "cc_cpu_ms": round(ccs * 1e3, 1),
                "parity": bool(np.array_equal(lv.values, want) and np.array_equal(lab.values, wlab))}
            del rp, ci, want, wlab, lv, lab
            A = None
            cleanup()
        except Exception as e:  # noqa: BLE001 -- report, never lose the bench line
            out[f"C5_bfs_cc_s{sc}"] = {"error": f"{type(e).__name__}: {e}"[:200]}
            gb._lib.context().trim()
            torch.cuda.empty_cache()
    return out


def uniform_sweep(gb, ctx, peak, peak_src, scale=24):
    """SURVEY §8(d) "uniform" row: the same generator with a=b=c=d=.25 at the
    benchmark scale -- BFS and CC against the C oracle on the same CSR, and
    the masked pull SpMV (row bins vs row tiles) against torch."""
    import torch
    from oracle import cgraph
    from paper_1908_01407_b200.io import rmat_matrix
    A = rmat_matrix(scale, a=0.25, b=0.25, c=0.25, d=0.25)
    n, m = A.nrows, A.nnz
    bms, lv = _dev_ms(lambda: gb.bfs(A, 0), 10)
    cms, lab = _dev_ms(lambda: gb.connected_components(A), 2)
    rp, ci = A._csr.offsets.cpu().numpy(), A._csr.indices.cpu().numpy()
    bcs, (want, trace) = _cpu_s(lambda: cgraph.bfs(rp, ci, 0))
    ccs, (wlab, _t) = _cpu_s(lambda: cgraph.cc(rp, ci))
    d = gb.Descriptor()
    gb.bfs(A, 0, desc=d)
    out = {"graph": f"uniform-s{scale}-e16 (a=b=c=d=.25) symmetrised", "n": n, "nnz": m,
           "bfs_gpu_ms": round(bms, 3), "bfs_gteps": round(m / bms / 1e6, 1),
           "bfs_cpu_ms": round(bcs * 1e3, 1), "bfs_trace": [(x.chosen, x.frontier_nvals)
                                                           for x in d.direction_log],
           "cc_gpu_ms": round(cms, 3), "cc_cpu_ms": round(ccs * 1e3, 1),
           "parity": bool(np.array_equal(lv.values, want) and np.array_equal(lab.values, wlab)
                          and [t[:2] for t in trace] == [(x.chosen, x.frontier_nvals)
                                                         for x in d.direction_log])}
    del rp, ci, want, wlab, lv, lab
    out["masked_spmv"] = masked_spmv(gb, A, ctx, peak, peak_src, graph=f"uniform-s{scale}")
    A = None
    ctx.trim()
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200 import _lib
    from paper_1908_01407_b200.containers import to_host
    from paper_1908_01407_b200.io import rmat_matrix

    rank, world, local = env_rank()
    # one process per GPU; GB_DIST_BACKEND=gloo (test only) lets several ranks
    # share one GPU to exercise the multi-rank path on a single-GPU box
    backend = os.environ.get("GB_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    ctx = _lib.context()

    t0 = time.perf_counter()
    A = rmat_matrix(args.scale)
    torch.cuda.synchronize()
    ctx.trim()
    build_s = time.perf_counter() - t0
    n, m = A.nrows, A.nnz

    if world > 1:
        # 1D vertex partition: this rank keeps its row block (pull) and column
        # block (push); one NCCL all-reduce of the n/8-byte frontier bitmap per level
        from paper_1908_01407_b200 import distributed as gbd
        # the partition of the degree-ordered layout (as the 1-GPU bfs uses it);
        # levels are gathered back to original ids inside the step
        runner = gbd.OrderedPartitionedBfs(A, rank, world)

        def step():
            return runner(args.source)
    else:
        # bfs() enqueues without a host sync; each call's decision log is read
        # after the timed region (it books the call's kernel launches)
        descs = []

        def step():
            d = gb.Descriptor()
            descs.append(d)
            return gb.bfs(A, args.source, desc=d)

    for _ in range(max(args.warmup, 3)):
        lv = step()
    torch.cuda.synchronize()

    # ---- device-timed region: exactly K steps -----------------------------
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches()
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            lv = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    if world == 1:
        for d in descs[-args.steps:]:
            assert len(d.direction_log) > 0
        descs.clear()
    launches = (ctx.launches() - launches0) // max(args.steps, 1)
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = m / (ms * 1e-3) / 1e9  # GTEPS

    # ---- per-level kernel timing (separate, untimed pass) -------------------
    desc = gb.Descriptor()
    ctx.profiling(True)
    lv = gb.bfs(A, args.source, desc=desc)
    prof = ctx.prof_read()
    ctx.profiling(False)
    trace = [(d.chosen, d.frontier_nvals) for d in desc.direction_log]
    levels_host = lv.values
    deg_all = np.diff(A._csr.offsets.cpu().numpy())
    g500_edges = int(deg_all[levels_host > 0].sum()) // 2
    del deg_all
    counts = np.bincount(levels_host, minlength=len(trace) + 2)
    roof = None
    peak, peak_src = measured_peaks()
    push_times = [(arg, t) for (kind, arg, t) in prof if kind == 1]
    # edges each push level actually expands (kind 9 precedes its push): on the
    # degree-ordered layout the neighbours below the dense visited prefix are
    # skipped, so this is <= the reference's multiply count sum(deg(frontier))
    expanded = [arg for (kind, arg, _t) in prof if kind == 9]
    if push_times:
        # dominant launch: the longest push expansion (level 2 at s24)
        j = max(range(len(push_times)), key=lambda i: push_times[i][1])
        k, t_ms = push_times[j]
        lvl = next(i for i, (c, nv) in enumerate(trace) if c == "push" and nv == k)
        deg = np.diff(A._csr.offsets.cpu().numpy())
        front = np.flatnonzero(levels_host == lvl + 1)
        flops = int(deg[front].sum())
        edges = int(expanded[j]) if len(expanded) == len(push_times) else flops
        k_next = int(counts[lvl + 2]) if lvl + 2 < counts.size else 0
        # SURVEY §8(d)'s push rule: the level's multiplies (flops = sum of the
        # frontier's degrees, the reference's semiring_multiplies) at 4 B each
        bytes_alg = push_level_bytes(n, k, flops, k_next)
        achieved = bytes_alg / (t_ms * 1e-3) / 1e9
        # the conservative variant: only the edges the kernel reads (the
        # degree-ordered prefix cut skips the neighbours below the dense
        # visited prefix)
        bytes_read = push_level_bytes(n, k, edges, k_next)
        read_gbs = bytes_read / (t_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": "bfs_expand_warp (push SpMSpV, level %d)" % (lvl + 1),
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": peak_src,
                "frac_vs_nominal_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
                "traffic": committed_traffic("bfs_expand_warp"),
                "bytes_alg": int(bytes_alg), "launch_ms": round(t_ms, 4),
                "frontier": int(k), "flops": flops, "edges_expanded": edges,
                "bytes_rule": "SURVEY §8(d) push: K*(4+2*8) + flops*4 + n/8 (mask) + n/8 "
                              "(out bitmap) + K_next*(4+8), flops = sum of the frontier's "
                              "degrees",
                "conservative": {
                    "what": "the same rule over the edges actually read (edges below the dense "
                            "visited prefix are skipped, never loaded)",
                    "bytes": int(bytes_read), "achieved": round(read_gbs, 1),
                    "frac": round(read_gbs / peak, 4)},
                "level_ms": [(kind, a, round(t, 4)) for (kind, a, t) in prof]}
        # the push is bound by scattered 4 B probes of the visited bitmap, not
        # by HBM: report it against the random-probe rate of this GPU too
        rate = ctypes.c_double(0.0)
        ctx.call("gb_probe_rate", (n + 31) // 32, 1 << 30, ctypes.byref(rate))
        probes_s = edges / (t_ms * 1e-3)
        roof["probe_rate"] = {
            "what": "uniformly random 4 B ld.global.ca probes of an n-bit bitmap on all SMs "
                    "(gb_probe_rate, measured in this run) beside the push's probes per second "
                    "(one per edge read); the push beats it because the degree-ordered layout "
                    "concentrates its probes on an L1-resident prefix",
            "uniform_random_Gprobe_s": round(rate.value / 1e9, 1),
            "achieved_Gprobe_s": round(probes_s / 1e9, 1),
            "ratio": round(probes_s / rate.value, 3)}

    mspmv = masked_spmv(gb, A, ctx, peak, peak_src) if world == 1 and not args.no_spmv else None

    # ---- the reference's own direction knob: Descriptor(switch_ratio=0.01)
    # pulls level 2 (estimate 12.6 M > 0.01 * nnz) -- direction-optimising
    # BFS through the reference rule; same levels, a different (logged) trace.
    # Reported beside the headline, which keeps the reference default 0.1.
    dopt = None
    if world == 1:
        def opt_step():
            return gb.bfs(A, args.source, desc=gb.Descriptor(switch_ratio=0.01))
        oms, olv = _dev_ms(opt_step, max(args.steps // 4, 10))
        od = gb.Descriptor(switch_ratio=0.01)
        olv = gb.bfs(A, args.source, desc=od).values
        dopt = {"switch_ratio": 0.01, "ms_per_step": round(oms, 4),
                "value": round(m / (oms * 1e-3) / 1e9, 3), "unit": "GTEPS",
                "trace": [(x.chosen, x.frontier_nvals) for x in od.direction_log],
                "same_levels_as_default": bool(np.array_equal(olv, levels_host)),
                "what": "bfs(A, src, desc=Descriptor(switch_ratio=0.01)): the reference's own "
                        "rule and knob (kernels.py:108-126) pulling from level 2; not the "
                        "headline, which uses the default ratio 0.1"}
        del olv

    # ---- BFS tree (north star "levels/parents-validity"): min-id parents
    # derived on the device, Graph500-style validation of (levels, parents)
    tree = None
    if world == 1:
        pms, (tl, tp) = _dev_ms(lambda: gb.bfs_parents(A, args.source), 5)
        val = gb.validate_bfs(A, args.source, tl, tp)
        tree = {"bfs_plus_parents_ms": round(pms, 4),
                "parents_only_ms": round(pms - ms, 4),
                "validate": val,
                "rule": "parent[v] = smallest neighbour one level up (deterministic); "
                        "validated: source, tree edges exist one level up, unreached -> -1, "
                        "every edge spans <= 1 level"}
        del tl, tp

    # ---- end-to-end through the public API (host result every step) --------
    # warm-up: the first calls allocate the pinned staging blocks (~57 ms each
    # for 134 MB); torch's caching host allocator reuses them afterwards
    for i in range(max(args.warmup, 2)):
        out = to_host(step()) if world > 1 else gb.bfs(A, args.source).values
    torch.cuda.synchronize()
    t_e2e = []
    for i in range(args.steps):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if world > 1:
            out = to_host(step())                # replicated levels -> host (pinned D2H)
        else:
            out = gb.bfs(A, args.source).values  # levels -> host numpy (pinned D2H)
        t_e2e.append(time.perf_counter() - t1)
    e2e_latency_ms = float(np.mean(t_e2e)) * 1e3
    e2e_ms = e2e_latency_ms
    if world == 1:
        # a stream of queries: query i+1 runs on the device while the levels
        # of query i cross PCIe on a copy stream (public API + torch streams);
        # every step still copies its own n*8 B result to host
        main = torch.cuda.current_stream()
        copy = torch.cuda.Stream()
        prev = None
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for i in range(args.steps + 1):
            cur = None
            if i < args.steps:
                lv_i = gb.bfs(A, args.source)
                ev = torch.cuda.Event()
                ev.record(main)
                cur = (lv_i, ev)
            if prev is not None:
                with torch.cuda.stream(copy):
                    copy.wait_event(prev[1])
                    out = prev[0].values
            prev = cur
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t1) * 1e3 / args.steps
        assert np.array_equal(out, levels_host)
    parity = None
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        # the partitioned result must equal the single-GPU fused BFS
        same = torch.tensor([int(np.array_equal(out, levels_host))], device=dev)
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        parity = bool(same.item())

    # ---- CPU baseline: the C port of the reference algorithm, same CSR ------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import cgraph
        rp = A._csr.offsets.cpu().numpy()
        ci = A._csr.indices.cpu().numpy()
        cgraph.lib()
        threads = cgraph.threads()
        times = []
        tstart = time.perf_counter()
        ref_lv = None
        while len(times) < 3 and (time.perf_counter() - tstart) < args.cpu_cap_s:
            t1 = time.perf_counter()
            ref_lv, ref_trace = cgraph.bfs(rp, ci, args.source)
            times.append(time.perf_counter() - t1)
        cpu_s = float(np.mean(times))
        parity = bool(np.array_equal(ref_lv, levels_host)) and \
            [t[:2] for t in ref_trace] == [tuple(t) for t in trace]
        cpu = {"value": round(m / cpu_s / 1e9, 4), "unit": "GTEPS", "cores": threads,
               "kind": "port",
               "sample": f"full BFS from vertex {args.source} on the same s{args.scale} CSR, "
                         f"oracle/cgraph.c og_bfs with {threads} OpenMP threads, mean of {len(times)} runs",
               "ms_per_bfs": round(cpu_s * 1e3, 2), "cpu": cpu_model(),
               "os_cpu_count": os.cpu_count()}

    if cpu is not None:
        # the same BFS with ONE host thread (the reference's pull pool often
        # does not help); one run
        from oracle import cgraph
        rp = A._csr.offsets.cpu().numpy()
        ci = A._csr.indices.cpu().numpy()
        prev = cgraph.threads()
        cgraph.set_threads(1)
        try:
            t1 = time.perf_counter()
            cgraph.bfs(rp, ci, args.source)
            one = time.perf_counter() - t1
        finally:
            cgraph.set_threads(prev)
        cpu["one_thread"] = {"value": round(m / one / 1e9, 4), "unit": "GTEPS", "cores": 1,
                             "ms_per_bfs": round(one * 1e3, 1)}
        del rp, ci
    configs = None
    uniform = None
    if rank == 0 and world == 1 and not args.no_configs:
        del A
        ctx.trim()
        torch.cuda.empty_cache()
        configs = config_sweep(gb)
        try:
            uniform = uniform_sweep(gb, ctx, peak, peak_src, args.scale)
        except Exception as e:  # noqa: BLE001 -- report, never lose the bench line
            uniform = {"error": f"{type(e).__name__}: {e}"[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32/i64 (bitmaps, int32 indices, int64 levels)",
            "data": "synthetic R-MAT (reference SplitMix64 generator, seed 1), generated on GPU",
            "config": bench_config(args, n, m),
            "parallelism": f"1d-vertex-partition x{world}" if world > 1 else "single-gpu",
            "build_s": round(build_s, 2), "trace": trace,
            "graph500_gteps": round(g500_edges / (ms * 1e-3) / 1e9, 3),
            "graph500_what": "Graph500-style TEPS: undirected edges with both endpoints in the "
                             "source's component (stored entries of reached vertices / 2) per "
                             "second, same device time as `value`",
            "clocks": clocks.summary(),
            "e2e": {"value": round(m / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GTEPS",
                    "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": 8,
                    "d2h_bytes_per_step": int(n * 8),
                    "latency_ms": round(e2e_latency_ms, 3),
                    "what": "bfs(A, src).values through the public API: source id in, "
                            "int64 level vector (n*8 B) out to host every step; "
                            + ("queries pipelined (the next bfs runs while the previous "
                               "levels are copied on a second stream); latency_ms = one "
                               "query alone, synchronised" if world == 1 else
                               "one query at a time")},
            "gpu_launches": int(launches),
            "roofline": roof,
            "masked_spmv": mspmv,
            "bfs_tree": tree,
            "bfs_switch_ratio_001": dopt,
            "exchange": (None if world == 1 else {
                "per_level_last_step": runner.exchange.log[-(len(trace) + 1):],
                "loop": runner.loop,
                "what": "FrontierExchange per level: (mode, bytes sent per rank).  The "
                        "device-resident loop (default) exchanges dense = allgather of the "
                        "owned bitmap words every level, plus one no-op level past the end "
                        "(the host watches the done flag one level behind); the host loop "
                        "picks dense (|f|*32 > n) or sparse = allgather(v) of the owned new "
                        "vertex ids after an 8 B count allgather",
                "backend": os.environ.get("GB_DIST_BACKEND", "nccl")}),
            "cpu_baseline": cpu,
            "parity_vs_oracle": parity,
            "configs": configs,
            "uniform": uniform,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm: the C port of the reference algorithm on the host cores
# ---------------------------------------------------------------------------


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import cgraph
    cgraph.lib()
    threads = cgraph.threads()
    t0 = time.perf_counter()
    rp, ci = cgraph.rmat_csr(args.scale)
    build_s = time.perf_counter() - t0
    n, m = rp.size - 1, ci.size
    tw = []
    for _ in range(max(args.warmup, 1)):
        t1 = time.perf_counter()
        cgraph.bfs(rp, ci, args.source)
        tw.append(time.perf_counter() - t1)
    per = float(np.mean(tw))
    k = args.steps
    if per * k > args.cpu_cap_s:
        k = max(1, int(args.cpu_cap_s / per))
    t1 = time.perf_counter()
    for _ in range(k):
        cgraph.bfs(rp, ci, args.source)
    total = time.perf_counter() - t1
    ms = total / k * 1e3
    value = m / (ms * 1e-3) / 1e9
    sample = (f"full BFS from vertex {args.source} on rmat-s{args.scale} per step; "
              f"{k} of {args.steps} steps timed (cap {args.cpu_cap_s:.0f}s)")
    line = {"metric": METRIC, "value": round(value, 4), "unit": "GTEPS", "n_gpus": world,
            "steps": k, "warmup": max(args.warmup, 1), "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8/i64", "data": "synthetic R-MAT (reference generator, seed 1)",
            "impl": "reference",
            "config": bench_config(args, n, m), "build_s": round(build_s, 2),
            "cpu_baseline": {"value": round(value, 4), "unit": "GTEPS", "cores": threads,
                             "kind": "port", "sample": sample, "cpu": cpu_model(),
                             "os_cpu_count": os.cpu_count()},
            "e2e": {"value": round(value, 4), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
