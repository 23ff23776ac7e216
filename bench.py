"""Benchmark of the RBF-FD hot path on B200 (BASELINE.json metric).

One step = the whole hot path over config C3 (3D unit cube, N = 1,000,000
uniform nodes, n = 35, PHS r^3 + degree-2 monomials, Laplacian):
    kNN stencils -> shape solve -> canonical CSR -> explicit Laplacian apply.

value      stencils/s through the step with inputs resident in HBM
           (device-timed with CUDA events, L2 flushed between steps)
e2e        same metric through the public API with host (pinned) inputs:
           positions + field H2D and the applied field D2H inside the region
           (wall clock, median of 3-5 steps; the per-step times are listed)
roofline   dominant kernel = the shape solve (fp64-pipe bound): algorithmic
           flops F = (2/3)s^3 + 2 r s^2 per stencil / its CUDA-event time,
           against the fp64 DFMA peak measured in this run; apply_roofline
           gives the Laplacian apply against MEASURED_PEAKS.json HBM GB/s
cpu_baseline  the C oracle (bit-exact restatement of the reference's numba
           kernel + kNN + CSR + matvec) on host cores over a bounded sample

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU (torchrun): ONE sharded problem of world x 1M nodes in
the unit cube (weak scaling: 1M targets per rank); positions replicated, each
rank selects stencils and solves shapes for its contiguous target block (no
collective), builds its CSR rows (global columns) and applies the Laplacian
after one NCCL all-gather of the field; value = all stencils / max-over-ranks
time.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

METRIC = "RBF-FD shapes/s (3D, n=35, deg-2 monomials); explicit Laplacian apply GB/s"
UNIT = "stencils/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="hybrid", choices=["hybrid", "replay", "fast"])
    ap.add_argument("--N", type=int, default=1_000_000)
    ap.add_argument("--cpu-sample", type=int, default=250_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the secondary C5 / C4-heat measurements")
    return ap.parse_args()


def c3_positions(N, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 1.0, (N, 3))


def flops_per_stencil(n, l, r):
    s = n + l
    return (2.0 / 3.0) * s**3 + 2.0 * r * s * s


def apply_bytes(N, nnz, r=1):
    return nnz * (8 * r + 4) + N * 8 + r * N * 8 + (N + 1) * 4


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture summary, else None."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            return int(json.load(f)[kernel]["bytes"])
    except (OSError, KeyError, ValueError):
        return None


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


_NVML_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("ready %d" % pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
while True:
    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    print("%d,%d" % (mhz, rs), flush=True)
    time.sleep(0.005)
"""


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region by a
    separate NVML process (5 ms; a thread would contend for the GIL with the
    launching thread), else an nvidia-smi -lms subprocess."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    NVML_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                 "hw_thermal_slowdown": 0x40}

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.kind = None
        self.max_mhz = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _NVML_SAMPLER, str(self.index)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            first = self.proc.stdout.readline()
            if first.startswith("ready"):
                self.max_mhz = float(first.split()[1])
                self.kind = "nvml"
                return self
            self.proc.kill()
            self.proc.wait()
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.kind = "nvidia-smi"
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], self.max_mhz, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            try:
                if self.kind == "nvml" and len(parts) == 2:
                    sm.append(float(parts[0]))
                    rs = int(parts[1])
                    reasons |= {nm for nm, bit in self.NVML_BITS.items() if rs & bit}
                elif len(parts) >= 6:
                    sm.append(float(parts[0]))
                    mx = float(parts[1])
                    reasons |= {nm for nm, flag in zip(names, parts[2:6]) if flag.lower() == "active"}
            except ValueError:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.kind}


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle (pinned bit-exact to the reference)
# ---------------------------------------------------------------------------

def cpu_pipeline_sample(pts, n, sample, threads=0):
    """Oracle kNN + weights + CSR + apply over `sample` targets; returns seconds."""
    import oracle

    N = pts.shape[0]
    targets = np.arange(0, N, max(1, N // sample), dtype=np.int64)[:sample]
    u = np.random.default_rng(1).standard_normal(N)
    t0 = time.perf_counter()
    st, _ = oracle.knn(pts, n, targets, threads=threads)
    w, fail, _ = oracle.phs_weights(pts, targets, st, ["laplacian"], degree=2, threads=threads)
    ip, ix, da = oracle.csr_canonical(targets, st, w[:, 0, :], N)
    oracle.apply(ip, ix, da, u, threads=1)
    return time.perf_counter() - t0, targets.shape[0]


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle

    pts = c3_positions(args.N, 0)
    cores = os.cpu_count() or 1
    oracle.build()
    for _ in range(args.warmup):
        cpu_pipeline_sample(pts, 35, max(1000, args.cpu_sample // 10), threads=cores)
    times, counts = [], []
    for _ in range(args.steps):
        dt, cnt = cpu_pipeline_sample(pts, 35, args.cpu_sample, threads=cores)
        times.append(dt)
        counts.append(cnt)
    value = sum(counts) / sum(times)
    sample = (f"C3 node set (N={args.N}); per step {args.cpu_sample} strided targets through oracle "
              f"kNN + shape solve + CSR + apply, {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": "C3", "N": args.N, "n": 35, "degree": 2,
                                        "families": ["laplacian"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1 or os.environ.get("MF_BENCH_SHARDED"):  # (the env switch runs the sharded path at N=1)
        return run_sharded(args, rank, world, local)

    import torch
    import torch.distributed as dist

    import paper_1912_13282_b200 as mf
    from paper_1912_13282_b200 import _lib, build as mfbuild
    from paper_1912_13282_b200.stencils import knn_device
    from paper_1912_13282_b200.storage import _structure_async, phs_weights_device, expand_families

    mfbuild.build()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    N, n, deg = args.N, 35, 2
    l = 10
    pts = c3_positions(N, rank)
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=deg, scale="support", solver="lu", mode=args.mode)
    fams = expand_families(["laplacian"], 3)
    u_host = np.random.default_rng(1).standard_normal(N)

    nodes = mf.NodeSet(pts, np.ones(N, dtype=np.int64))
    pos_d = nodes.positions_device()
    u_d = torch.from_numpy(u_host).to(dev)
    all_idx = np.arange(N, dtype=np.int64)
    rows_d = torch.arange(N, dtype=torch.int64, device=dev)  # targets = pool = rows, resident
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    # setup: prime the caching allocator with one segment larger than a step's
    # working set (~2 GB at C3), so steps carve their buffers from it instead of
    # calling cudaMalloc while the clock runs
    _prime = torch.empty(8 << 30, dtype=torch.uint8, device=dev)
    del _prime

    host_marks = []

    su = torch.empty(N, dtype=torch.float64, device=dev)
    sy = torch.empty(N, dtype=torch.float64, device=dev)
    kernel_timers = []

    def step(timers=None):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if timers is not None else None
        kev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if timers is not None else None
        hm = [time.perf_counter()]
        if ev:
            ev[0].record(stream)
        st, _ = knn_device(nodes, n, rows_d, rows_d)
        hm.append(time.perf_counter())
        if ev:
            ev[1].record(stream)
        # (as compute_weights: CSR structure + locality order on the side stream,
        # overlapping the shape solve's re-solve pass)
        pre = _structure_async(N, rows_d, st, n, pos_d)
        w, status, first_fail, n_rep = phs_weights_device(pos_d, rows_d, st, eng, fams, 3)
        hm.append(time.perf_counter())
        if ev:
            ev[2].record(stream)
        store = mf.WeightStore(N, all_idx, st, {"laplacian": w[:, 0, :]}, n, rows_d=rows_d, positions_d=pos_d)
        store._adopt_structure(*pre)
        mat = store.matrix("laplacian")
        order_p, idx_p, val_p, len_p = mat.plan_direct()
        hm.append(time.perf_counter())
        if ev:
            ev[3].record(stream)
        # mat.apply_device(u_d), spelled out through the C ABI so the apply kernel
        # is bracketed by events: one launch (Morton-row plan, node-numbered
        # columns: the field is read in place, the result scattered by the kernel)
        y = torch.empty(N, dtype=torch.float64, device=dev)
        if ev:
            kev[0].record(stream)
        _lib.check(lib.mf_plan_apply_direct(idx_p.data_ptr(), val_p.data_ptr(), len_p.data_ptr(), N, n,
                                            order_p.data_ptr(), u_d.data_ptr(), y.data_ptr(), _lib.stream_ptr()),
                   "mf_plan_apply_direct")
        if ev:
            kev[1].record(stream)
        hm.append(time.perf_counter())
        if ev:
            ev[4].record(stream)
            timers.append(ev)
            kernel_timers.append(kev)
            host_marks.append(np.diff(hm) * 1e3)
        return y, first_fail, n_rep

    for _ in range(args.warmup):
        y, ff, _ = step()
    torch.cuda.synchronize()
    if os.environ.get("MF_BENCH_DEBUG"):
        # host-side stage times with a synchronize after each stage (diagnostics only)
        import time as _t
        marks = []
        t0 = _t.perf_counter()
        st_, _ = knn_device(nodes, n, rows_d, rows_d); torch.cuda.synchronize(); marks.append(_t.perf_counter())
        w_, *_ = phs_weights_device(pos_d, rows_d, st_, eng, fams, 3); torch.cuda.synchronize(); marks.append(_t.perf_counter())
        store_ = mf.WeightStore(N, all_idx, st_, {"laplacian": w_[:, 0, :]}, n, rows_d=rows_d, positions_d=pos_d)
        mat_ = store_.matrix("laplacian"); torch.cuda.synchronize(); marks.append(_t.perf_counter())
        mat_.plan(True); torch.cuda.synchronize(); marks.append(_t.perf_counter())
        mat_.apply_device(u_d); torch.cuda.synchronize(); marks.append(_t.perf_counter())
        names = ["knn", "phs", "csr", "plan", "apply"]
        prev = t0
        for nm_, mk in zip(names, marks):
            print(f"[debug] {nm_}: {1e3 * (mk - prev):.2f} ms", file=sys.stderr)
            prev = mk
    assert int(ff.item()) == _lib.SENTINEL_OK, "shape solve reported a failing stencil"

    # fp64 pipe peak for the roofline denominator (measured in this run)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    probe_out = torch.empty(1, dtype=torch.float64, device=dev)
    fl = ctypes_double()
    for _ in range(2):
        lib.mf_dfma_probe(sms * 8, 256, 2000, probe_out.data_ptr(), _lib.stream_ptr(), fl)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    lib.mf_dfma_probe(sms * 8, 256, 2000, probe_out.data_ptr(), _lib.stream_ptr(), fl)
    e1.record(stream)
    torch.cuda.synchronize()
    fp64_peak = fl.value / (e0.elapsed_time(e1) * 1e-3) / 1e12

    # ---- stage breakdown: eager steps, events between the stages (host enqueue
    # times recorded alongside; a stage whose host side stalls longer than the
    # device work queued ahead of it would show the stall here)
    gc.collect()
    gc.disable()
    timers = []
    for _ in range(args.steps):
        flush.zero_()
        y, ff, n_rep = step(timers)
    torch.cuda.synchronize()
    stage = np.array([[a.elapsed_time(b) for a, b in zip(ev[:-1], ev[1:])] for ev in timers])  # ms
    host_ms = np.array(host_marks[-args.steps:])

    # ---- timed region: the same step captured once as a CUDA graph and replayed
    # K times (no host work between kernels, so host stalls cannot leak into the
    # device time); events around each replay, L2 flushed between replays
    # (outside the events)
    launches0 = lib.mf_launch_count()
    graph = torch.cuda.CUDAGraph()
    cap_stream = torch.cuda.Stream()
    cap_stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap_stream):
        with torch.cuda.graph(graph, stream=cap_stream):
            g_out = step()
    torch.cuda.current_stream().wait_stream(cap_stream)
    launches = lib.mf_launch_count() - launches0  # our kernels per step (captured once)
    graph.replay()
    torch.cuda.synchronize()
    assert int(g_out[1].item()) == _lib.SENTINEL_OK, "shape solve reported a failing stencil (graph)"
    assert torch.equal(g_out[0], y), "graph replay differs from the eager step"
    ev_pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for e0, e1 in ev_pairs:
            flush.zero_()
            e0.record(stream)
            graph.replay()
            e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gc.enable()
    step_list = [a.elapsed_time(b) for a, b in ev_pairs]
    if os.environ.get("MF_BENCH_DEBUG"):
        print("[debug] per-step stage ms (knn, shape, csr+plan, apply):\n" + np.array2string(stage, precision=2),
              file=sys.stderr)
        print("[debug] per-step host ms to enqueue each stage:\n" + np.array2string(host_ms, precision=2),
              file=sys.stderr)
        print("[debug] graph steps ms: " + " ".join(f"{t:.3f}" for t in step_list), file=sys.stderr)
    step_ms = float(np.mean(step_list))
    t_local = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    step_ms_max = float(t_local.item())
    value = world * N / (step_ms_max * 1e-3)
    n_replayed = int(g_out[2].item())

    # median over the eager steps: one host hiccup (an eager step that waits on the host
    # mid-stage) must not leak into the stage times the rooflines are computed from
    knn_ms, phs_ms, csr_ms, apply_ms = (float(x) for x in np.median(stage, axis=0))
    F = flops_per_stencil(n, l, 1)
    phs_tflops = N * F / (phs_ms * 1e-3) / 1e12
    nnz = N * n
    b_apply = apply_bytes(N, nnz)
    apply_gbs = b_apply / (apply_ms * 1e-3) / 1e9
    ell_ms = float(np.mean([a.elapsed_time(b) for a, b in kernel_timers]))
    ell_gbs = b_apply / (ell_ms * 1e-3) / 1e9
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        pts_pin = torch.empty((N, 3), dtype=torch.float64, pin_memory=True).numpy()
        pts_pin[:] = pts
        u_pin = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
        u_pin[:] = u_host
        types = np.ones(N, dtype=np.int64)

        def e2e_step():
            nodes_h = mf.NodeSet(pts_pin, types)
            nodes_h = mf.find_closest_stencils(nodes_h, n)
            store_h = mf.compute_weights(nodes_h, eng, ["laplacian"])
            return store_h.apply_all("laplacian", u_pin)

        e2e_step()
        e2e_step()
        torch.cuda.synchronize()
        gc.collect()
        gc.disable()
        ts = []
        for _ in range(max(5, min(args.steps, 10))):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            y_h = e2e_step()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        gc.enable()
        # median step: host-side hiccups (allocator, GC) hit single wall-clock steps
        e2e_t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e = {"value": world * N / float(e2e_t.item()), "unit": UNIT,
               # positions and field (whole-set selections send no index arrays)
               "h2d_bytes_per_step": int(pts.nbytes + u_host.nbytes),
               "d2h_bytes_per_step": int(y_h.nbytes), "stat": f"median of {len(ts)} wall-clock steps",
               "steps_ms": [round(1e3 * t, 3) for t in ts]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        oracle.build()
        cores = os.cpu_count() or 1
        cpu_pipeline_sample(pts, n, 20_000, threads=cores)
        secs, cnt = cpu_pipeline_sample(pts, n, args.cpu_sample, threads=cores)
        cpu = {"value": cnt / secs, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{cnt} strided C3 targets through oracle kNN + shape solve + CSR + apply "
                         f"({secs:.2f} s, {cores} threads)"}

    c5 = c4 = None
    if rank == 0 and world == 1 and not args.no_c5:
        c4 = measure_c4_heat(mf, dev, hbm_peak)
        c5 = measure_c5(mf, lib, dev, fp64_peak, hbm_peak)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3", "N": N, "n": n, "degree": deg, "families": ["laplacian"],
                       "shape_mode": args.mode, "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"weak x{world} (independent node sets per rank)"},
            "stage_ms": {"knn": knn_ms, "shape_solve": phs_ms, "csr_and_plan": csr_ms, "apply": apply_ms},
            "shapes_per_s": N / (phs_ms * 1e-3),
            "apply_gbs": apply_gbs,
            "roofline": {"bound": "fp64", "kernel": "mf_phs_weights (shape solve)",
                         "achieved": phs_tflops, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": phs_tflops / fp64_peak, "traffic": ncu_traffic("phs_ns2"),
                         "note": "F=(2/3)s^3+2rs^2 per stencil (s=45, r=1); peak = DFMA probe measured "
                                 "in this run (MEASURED_PEAKS.json has no fp64 entry)"},
            "apply_roofline": {"bound": "hbm", "kernel": "plan_apply_direct_k (Morton-ordered ELL-32 row sums, node-numbered columns, result scattered in-kernel)",
                               "achieved": ell_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": ell_gbs / hbm_peak,
                               "kernel_ms": ell_ms, "stage_gbs": apply_gbs,
                               "traffic": ncu_traffic("plan_apply_direct_k"), "bytes_per_launch": b_apply,
                               "note": "peak = MEASURED_PEAKS.json hbm_gbs (of measured)"},
            "knn_roofline": {"bound": "latency/issue (reported against HBM)", "kernel": "mf_knn (fast passes + fallback)",
                             "achieved": (N * 3 * 8 + N * n * 4) / (knn_ms * 1e-3) / 1e9, "peak": hbm_peak,
                             "unit": "GB/s", "frac": (N * 3 * 8 + N * n * 4) / (knn_ms * 1e-3) / 1e9 / hbm_peak,
                             "traffic": ncu_traffic("knn_fast"),
                             "note": "B_knn = N*d*8 + T*n*4 (SURVEY 8d); the search is bound by dependent "
                                     "loads and issue, not by these bytes"},
            "replayed_stencils": n_replayed,
            "gpu_launches": int(launches),
            "timing": {"value_from": f"{args.steps} replays of the step captured as one CUDA graph "
                                     "(device events around each replay, L2 flushed between)",
                       "steps_ms": [round(t, 4) for t in step_list],
                       "spread": (max(step_list) - min(step_list)) / float(np.median(step_list)),
                       "eager_ms_per_step": float(stage.sum(axis=1).mean()),
                       "eager_steps_ms": [round(float(t), 4) for t in stage.sum(axis=1)],
                       "eager_host_enqueue_ms": [round(float(t), 3) for t in host_ms.sum(axis=1)],
                       "stage_ms_from": "median over the eager steps, events between stages"},
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "secondary": {"C5": c5, "C4_heat": c4},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_c5(mf, lib, dev, fp64_peak, hbm_peak):
    """Config C5 (3D ball, N = 4M, n = 70, degree 4, laplacian + gradient) once
    through the same stages (not part of the headline value): stage times with
    CUDA events after one warm-up pass, the shape-solve roofline and the
    one-pass four-family apply against HBM."""
    import torch

    from paper_1912_13282_b200 import workloads

    w = workloads.c5()
    nodes = mf.NodeSet(w.positions, w.types)
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu")
    u = torch.from_numpy(w.field).to(dev)
    stream = torch.cuda.current_stream()
    res = None
    for it in range(2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream)
        nd = mf.find_closest_stencils(nodes, w.n)
        ev[1].record(stream)
        store = mf.compute_weights(nd, eng, w.families)
        ev[2].record(stream)
        keys = store.families
        for k in keys:
            store.matrix(k).plan(True)
        ev[3].record(stream)
        ys = store.apply_families(keys, u)
        ev[4].record(stream)
        torch.cuda.synchronize()
        res = [a.elapsed_time(b) for a, b in zip(ev[:-1], ev[1:])]
        del store, nd, ys  # (the measured pass reuses the warm-up pass's cached blocks: no cudaMalloc in the stages)
    torch.cuda.empty_cache()
    knn_ms, shape_ms, plan_ms, apply_ms = res
    n, l, r = w.n, 35, len(keys)
    s_ = n + l
    F = (2.0 / 3.0) * s_ ** 3 + 2.0 * r * s_ * s_
    tflops = w.N * F / (shape_ms * 1e-3) / 1e12
    nnz = w.N * n
    b_apply = nnz * (8 * r + 4) + w.N * 8 + r * w.N * 8 + (w.N + 1) * 4
    return {"workload": "C5: 3D ball, N=4,000,000, n=70, degree 4, laplacian + gradient (4 families)",
            "stage_ms": {"knn": knn_ms, "shape_solve": shape_ms, "csr_and_plans": plan_ms,
                         "apply_4_families_one_pass": apply_ms},
            "stencils_per_s_through_step": w.N / (sum(res) * 1e-3),
            "shape_roofline": {"bound": "fp64", "achieved": tflops, "peak": fp64_peak, "unit": "TFLOP/s",
                               "frac": tflops / fp64_peak, "note": "F = (2/3)s^3 + 2rs^2, s = 105, r = 4"},
            "apply_roofline": {"bound": "hbm", "achieved": b_apply / (apply_ms * 1e-3) / 1e9, "peak": hbm_peak,
                               "unit": "GB/s", "frac": b_apply / (apply_ms * 1e-3) / 1e9 / hbm_peak,
                               "bytes": b_apply, "note": "stage incl. the field permutes (u gather, y scatters)"},
            "timing": "one pass after one warm-up pass, CUDA events; not part of value"}


def measure_c4_heat(mf, dev, hbm_peak):
    """Config C4 (2D unit square, N = 1M, n = 15): 1000 forward-Euler heat steps on the
    resident store at the stable dt = 0.1 h_min^2 (variant 4b), best of
    three run_heat_explicit calls after a short warm-up; not part of the headline value."""
    import torch

    from paper_1912_13282_b200 import workloads

    w = workloads.make("C4")
    nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n)
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu")
    store = mf.compute_weights(nodes, eng, w.families)
    st = nodes.stencil_matrix_device(np.arange(w.N)).cpu().numpy()
    dd = w.positions[st[:, 1]] - w.positions
    hmin = float(np.sqrt(np.min(np.einsum("ij,ij->i", dd, dd))))
    dt = 0.1 * hmin * hmin
    steps = 1000
    mf.run_heat_explicit(nodes, store, dt=dt, steps=5, dirichlet={-1: 0.0}, initial=w.field, return_device=True)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        u = mf.run_heat_explicit(nodes, store, dt=dt, steps=steps, dirichlet={-1: 0.0}, initial=w.field,
                                 return_device=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ok = bool(torch.isfinite(u).all().item())
    t = min(ts)
    nnz = w.N * w.n
    b_step = nnz * 12 + w.N * 8 + w.N * 8 + (w.N + 1) * 4 + w.N  # B_apply(r = 1) + N
    gbs = steps * b_step / (t * 1e-3) / 1e9
    del store, nodes
    torch.cuda.empty_cache()
    return {"workload": "C4: 2D unit square, N=1,000,000, n=15, 1000 forward-Euler steps, dt = 0.1 h_min^2",
            "heat_1000_steps_ms": t, "calls_ms": [round(x, 3) for x in ts], "us_per_step": 1e3 * t / steps,
            "finite": ok, "dt": dt,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                         "bytes_per_step": b_step,
                         "note": "algorithmic B_heat per step; the packed operator reads less (DESIGN 3)"},
            "timing": "run_heat_explicit(..., return_device=True) from a host initial field, CUDA events; "
                      "includes the operator packing and the field upload of each call"}


def run_sharded(args, rank, world, local):
    """One C3-density problem of world x N nodes, targets sharded over the ranks."""
    import torch
    import torch.distributed as dist

    import paper_1912_13282_b200 as mf
    from paper_1912_13282_b200 import _lib, build as mfbuild
    from paper_1912_13282_b200.parallel import RowPartition, ShardedProblem, allgather_field
    from paper_1912_13282_b200.stencils import knn_device
    from paper_1912_13282_b200.storage import expand_families, phs_weights_device

    mfbuild.build()
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    N = world * args.N
    n, deg = 35, 2
    # the same node set on every rank (positions replicated, 24 MB per 1M nodes)
    pts = np.random.default_rng(0).uniform(0.0, 1.0, (N, 3))
    part = RowPartition(N, world, rank)
    lo, hi = part.lo, part.hi
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=deg, scale="support", solver="lu", mode=args.mode)
    fams = expand_families(["laplacian"], 3)
    u_host = np.random.default_rng(1).standard_normal(N)
    nodes = mf.NodeSet(pts, np.ones(N, dtype=np.int64))
    pos_d = nodes.positions_device()
    tg_host = np.arange(lo, hi, dtype=np.int64)
    tg_d = torch.arange(lo, hi, dtype=torch.int64, device=dev)
    pool_d = torch.arange(N, dtype=torch.int64, device=dev)
    u_loc = torch.from_numpy(u_host[lo:hi]).to(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        st, _ = knn_device(nodes, n, tg_d, pool_d)
        if ev:
            ev[1].record(stream)
        w, _, first_fail, _ = phs_weights_device(pos_d, tg_d, st, eng, fams, 3)
        if ev:
            ev[2].record(stream)
        store = mf.WeightStore(N, tg_host, st, {"laplacian": w[:, 0, :]}, n, rows_d=tg_d, positions_d=pos_d)
        mat = store.matrix("laplacian")
        if ev:
            ev[3].record(stream)
        u_full = allgather_field(u_loc, part)  # NCCL all-gather of the field blocks
        y = torch.empty(hi - lo, dtype=torch.float64, device=dev)
        _lib.check(lib.mf_apply(mat.indptr_device[lo:].data_ptr(), mat.indices_device.data_ptr(),
                                mat.data_device.data_ptr(), u_full.data_ptr(), y.data_ptr(), hi - lo,
                                _lib.stream_ptr()), "mf_apply")
        if ev:
            ev[4].record(stream)
        return y, first_fail

    for _ in range(args.warmup):
        y, ff = step()
    torch.cuda.synchronize()
    assert int(ff.item()) == _lib.SENTINEL_OK, "shape solve reported a failing stencil"
    gc.collect()
    gc.disable()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    launches0 = lib.mf_launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for ev in evs:
            flush.zero_()
            step(ev)
        torch.cuda.synchronize()
    dist.barrier()
    gc.enable()
    launches = (lib.mf_launch_count() - launches0) / max(args.steps, 1)
    stage = np.array([[a.elapsed_time(b) for a, b in zip(ev[:-1], ev[1:])] for ev in evs])
    step_list = stage.sum(axis=1)
    t_local = torch.tensor([float(np.mean(step_list))], dtype=torch.float64, device=dev)
    dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    step_ms_max = float(t_local.item())
    value = N / (step_ms_max * 1e-3)

    # e2e through the public sharded API: host positions and field block in,
    # the rank's applied block out
    e2e = None
    if not args.no_e2e:
        ts = []
        for it in range(4):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sh = ShardedProblem(mf.NodeSet(pts, np.ones(N, dtype=np.int64)), n, eng, ["laplacian"], part=part)
            yb = sh.apply_all("laplacian", torch.from_numpy(u_host[lo:hi]).to(dev)).cpu().numpy()
            torch.cuda.synchronize()
            if it:
                ts.append(time.perf_counter() - t0)
        e2e_t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e = {"value": N / float(e2e_t.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(pts.nbytes + 8 * (hi - lo)), "d2h_bytes_per_step": int(yb.nbytes),
               "stat": f"median of {len(ts)} wall-clock steps, max over ranks"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3-density sharded", "N": N, "n": n, "degree": deg, "families": ["laplacian"],
                       "shape_mode": args.mode, "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"sharded x{world}: one {N}-node problem, contiguous target blocks, "
                                      "positions replicated, one NCCL all-gather of the field per apply"},
            "stage_ms": dict(zip(["knn", "shape_solve", "csr", "allgather_and_apply"],
                                 [float(x) for x in stage.mean(axis=0)])),
            "gpu_launches": int(launches),
            "timing": {"value_from": f"{args.steps} eager steps, device events, max over ranks",
                       "steps_ms": [round(float(t), 4) for t in step_list]},
            "clocks": clocks.summary(),
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def ctypes_double():
    import ctypes

    return ctypes.c_double(0.0)


if __name__ == "__main__":
    main()
