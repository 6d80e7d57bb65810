#!/usr/bin/env python3
"""Benchmark of the hybrid AMF + W1 Wiener hot path (BASELINE.json metric) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

A step is one pass of the hot path over one batch of synthetic input: one phantom image of the
chosen BASELINE.json config (default config 1, 1600x1600), or for config 3 the 512-slice stack.
``value`` = whole-job MPix/s with inputs resident in HBM (a rotating set of input/output buffers
larger than L2, so every step reads cold data); ``e2e`` = the same metric through the C ABI with
pinned HOST buffers (H2D copy, kernels, D2H copy inside the timed region).  N > 1 runs under
torchrun, one process per GPU: strips with NCCL halo exchange + one allreduce (strip configs,
strong scaling), or slice sharding (config 3, weak scaling).  ``--impl reference`` times the
reference's own CPU AMF (oracle/_ref, compiled from the reference sources) plus the W1 oracle on
all host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPix/s for hybrid AMF+Wiener (uint8) at 1/2/4/8 B200; % of roofline"
L2_BYTES = 126 * 1024 * 1024


def load_counters(cfg):
    """Per-launch ncu counters committed under profiles/ (profiles/ncu_counters.json, from one
    ncu --set full capture per config): DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and
    warp instructions (smsp__inst_executed.sum) of each stage -- measured once, reported beside the
    live timings (`traffic`, and the instruction-issue roofline)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_counters.json")) as f:
            return json.load(f).get(f"config{cfg}", {})
    except Exception:
        return {}


def issue_roofline(kernel, counters, ms, sm_mhz):
    """Warp-instruction issue rate of a stage vs the B200 peak (148 SMs x 4 schedulers x 1 / clk)."""
    c = counters.get(kernel)
    if not c or not ms or not sm_mhz:
        return None
    ach = c["warp_instr"] / (ms * 1e-3) / 1e9
    peak = 148 * 4 * sm_mhz * 1e6 / 1e9
    return {"bound": "issue", "kernel": kernel, "achieved": round(ach, 1), "peak": round(peak, 1),
            "unit": "G warp-instr/s", "frac": round(ach / peak, 4),
            "source": "warp instructions per launch from profiles/ncu_counters.json, duration live"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _sample(self):
        clk = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
        mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.samples.append(clk)
        for bit, name in self.REASONS.items():
            if mask & bit and name != "gpu_idle":
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()
            if not self.samples:
                try:
                    self._sample()
                except Exception:
                    pass

    def report(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_reference(cfg, c, threads, seconds, gpu_pixels_fn=None):
    """Reference AMF (adaptive_median_parallel, parts = workers = threads, compiled from the
    reference sources in oracle/_ref) + W1 oracle on `threads` row bands, repeated on the
    config's image until `seconds` of CPU work (a bounded sample)."""
    import oracle
    from paper_2005_05371_b200 import capi
    kind = "reference" if oracle.ref_available() else "port"
    rows, cols = c["rows"], c["cols"]
    img = capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], 0)
    done_px, t_total, reps = 0, 0.0, 0
    while reps == 0 or (t_total < seconds and reps < 50):
        if kind == "reference":
            _, ta, tw = oracle.ref_hybrid_baseline(img, c["smax"], c["win"], threads)
            t_total += ta + tw
        else:
            t0 = time.perf_counter()
            oracle.hybrid(img, c["smax"], c["win"])
            t_total += time.perf_counter() - t0
        done_px += rows * cols
        reps += 1
    sample = (f"{reps} x {rows}x{cols} config-{cfg} phantom (seed 0); AMF = reference "
              f"adaptive_median_parallel (parts=workers={threads}), Wiener = W1 oracle on {threads} threads "
              "(the reference has no local Wiener)") if kind == "reference" else \
        f"{reps} x {rows}x{cols} config-{cfg} phantom, W1+AMF oracle port, 1 thread"
    return {"value": done_px / t_total / 1e6, "unit": "MPix/s", "cores": threads if kind == "reference" else 1,
            "kind": kind, "sample": sample, "seconds": round(t_total, 3)}


def run_reference(args, cfg, c):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    # each step: a bounded sample of the workload (one image) on all host cores
    per_step = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference(cfg, c, threads, seconds=0.0)
        if i >= args.warmup:
            per_step.append(r)
    value = sum(r["value"] for r in per_step) / len(per_step)
    r0 = per_step[0]
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "MPix/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(c["rows"] * c["cols"] / value / 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload(cfg, c, 1),
        "cpu_baseline": {"value": round(value, 3), "unit": "MPix/s", "cores": r0["cores"], "kind": r0["kind"],
                         "sample": r0["sample"]},
        "e2e": {"value": round(value, 3), "unit": "MPix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload(cfg, c, n, exclusive=True):
    slices = c["slices"]
    d = {"workload": f"config{cfg}: {c['rows']}x{c['cols']} uint8 phantom"
         + (f" x {slices} slices" if slices > 1 else "")
         + f", {c['ellipses']} ellipses, sigma {c['sigma']}, S&P {c['density']}, AMF Smax {c['smax']}, "
           f"Wiener {c['win']}x{c['win']}",
         "pixels_per_step": c["rows"] * c["cols"] * slices,
         "partition": (f"{n} slice shards" if slices > 1 else f"{n} horizontal strips") if n > 1 else "1 GPU",
         "l2": "rotating input/output buffers > 3x L2 (cold reads every step)",
         "device_mode": "exclusive (hyb_set_exclusive: plain persistent launches)" if exclusive
         else "shared (cooperative launches)"}
    return d


def run_gpu(args, cfg, c):
    import torch
    import torch.distributed as dist

    from paper_2005_05371_b200 import capi
    from paper_2005_05371_b200.partition import CudaStripBackend, StripPlan, hybrid_strip_step

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    # a dedicated stream: the legacy default stream's handle is 0, which the C ABI reads as
    # "use the context's own stream"
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = capi.Context(local)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_exclusive(not args.shared_gpu)  # the bench owns the GPU (dedicated-device mode)
    lib = capi.lib

    rows, cols, slices = c["rows"], c["cols"], c["slices"]
    smax, win = c["smax"], c["win"]
    hbm, hbm_src = peaks()

    # ---------------- inputs (host phantom -> HBM) ----------------
    if slices > 1:
        my = [s for s in range(slices) if s % world == rank]
        host = torch.from_numpy(__import__("numpy").stack(
            [capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], s) for s in my]))
        unit_bytes = host.numel()
    else:
        img = torch.from_numpy(capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], 0))
        if world > 1:
            plan = StripPlan(rows, cols, smax, win, world, rank)
            host = img[plan.g_slice()].contiguous()
        else:
            host = img
        unit_bytes = host.numel()
    nbuf = max(1, math.ceil(3 * L2_BYTES / (2 * unit_bytes)))
    g_bufs = [host.to(dev) for _ in range(nbuf)]
    y_bufs = [torch.empty_like(g) if slices > 1 or world == 1 else
              torch.empty((plan.core, cols), dtype=torch.uint8, device=dev) for g in g_bufs]

    if slices == 1 and world > 1:
        backend = CudaStripBackend(ctx)
        f_strip = torch.empty((plan.f_rows, cols), dtype=torch.uint8, device=dev)
        w_dev = torch.zeros(1, dtype=torch.int64, device=dev)

    def step(i):
        g, y = g_bufs[i % nbuf], y_bufs[i % nbuf]
        if slices > 1:
            capi.check(lib.hyb_hybrid_batch_u8(ctx.ptr, g.data_ptr(), cols, rows * cols, g.shape[0], rows, cols,
                                               smax, win, y.data_ptr(), cols, rows * cols, None), ctx.ptr)
        elif world == 1:
            capi.check(lib.hyb_hybrid_u8(ctx.ptr, g.data_ptr(), cols, rows, cols, smax, win, 1, y.data_ptr(), cols,
                                         None), ctx.ptr)
        else:
            hybrid_strip_step(backend, plan, g, f_strip, y, w_dev)

    def timed(fn, k):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(k):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # untimed warm-up: at least W steps and two passes over the rotating buffers (the library
    # captures a CUDA graph per buffer pair on its second use and replays it afterwards)
    for i in range(max(args.warmup, 2 * nbuf)):
        step(i)
    torch.cuda.synchronize()
    l0 = ctx.launches()
    with ClockSampler(local) as clk:
        ms = timed(step, args.steps)
    launches = ctx.launches() - l0
    px_total = rows * cols * slices
    ms_step = ms / args.steps
    value = px_total / (ms_step * 1e-3) / 1e6

    # ---------------- per-kernel breakdown (same inputs, CUDA events on the launch stream) --------
    kern = {}
    if world == 1:
        f_scr = [torch.empty_like(g) for g in g_bufs]
        nsl = g_bufs[0].shape[0] if slices > 1 else 1

        def amf_only(i):
            g, f = g_bufs[i % nbuf], f_scr[i % nbuf]
            if slices > 1:
                capi.check(lib.hyb_amf_batch_u8(ctx.ptr, g.data_ptr(), cols, rows * cols, nsl, rows, cols, smax,
                                                f.data_ptr(), cols, rows * cols), ctx.ptr)
            else:
                capi.check(lib.hyb_amf_u8(ctx.ptr, g.data_ptr(), cols, rows, cols, 0, rows, smax, f.data_ptr(), cols,
                                          None, cols), ctx.ptr)

        for i in range(3):
            amf_only(i)
        k_amf = max(args.steps, 10)
        t_amf = timed(amf_only, k_amf) / k_amf
        # the two Wiener launches (stats + gain) on the AMF outputs
        w_dev1 = torch.zeros(max(nsl, 1), dtype=torch.int64, device=dev)

        def wiener_only(i):
            f, y = f_scr[i % nbuf], y_bufs[i % nbuf]
            if slices > 1:
                capi.check(lib.hyb_hybrid_batch_u8(ctx.ptr, f.data_ptr(), cols, rows * cols, nsl, rows, cols, 3, win,
                                                   y.data_ptr(), cols, rows * cols, None), ctx.ptr)
            else:
                capi.check(lib.hyb_wiener_stats_u8(ctx.ptr, f.data_ptr(), cols, rows, cols, 0, rows, win,
                                                   w_dev1.data_ptr()), ctx.ptr)
                capi.check(lib.hyb_wiener_gain_u8(ctx.ptr, f.data_ptr(), cols, rows, cols, 0, rows, win,
                                                  w_dev1.data_ptr(), rows * cols, y.data_ptr(), cols), ctx.ptr)

        t_w = None
        if slices == 1:
            for i in range(3):
                wiener_only(i)
            t_w = timed(wiener_only, k_amf) / k_amf
        kern = {"amf_ms": round(t_amf, 4), "wiener_ms": round(t_w, 4) if t_w else None}

    # ---------------- e2e through the C ABI with pinned host buffers ----------------
    e2e = None
    if world == 1:
        h_in = host.pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()

        def e2e_step(i):
            if slices > 1:
                capi.check(lib.hyb_hybrid_batch_u8(ctx.ptr, h_in.data_ptr(), cols, rows * cols, h_in.shape[0], rows,
                                                   cols, smax, win, h_out.data_ptr(), cols, rows * cols, None),
                           ctx.ptr)
            else:
                capi.check(lib.hyb_hybrid_u8(ctx.ptr, h_in.data_ptr(), cols, rows, cols, smax, win, 1,
                                             h_out.data_ptr(), cols, None), ctx.ptr)

        for i in range(max(2, args.warmup)):
            e2e_step(i)
        k_e2e = max(1, args.steps)  # the same K as the device-resident loop
        t0 = time.perf_counter()
        ms_e2e = timed(e2e_step, k_e2e)
        wall = (time.perf_counter() - t0) / k_e2e
        e2e = {"value": round(px_total / (ms_e2e / k_e2e * 1e-3) / 1e6, 3), "unit": "MPix/s",
               "h2d_bytes_per_step": int(h_in.numel()), "d2h_bytes_per_step": int(h_out.numel()),
               "ms_per_step": round(ms_e2e / k_e2e, 4), "wall_ms_per_step": round(wall * 1e3, 4)}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---------------- roofline of the dominant kernel ----------------
    roofline = None
    fused = world == 1 and launches == args.steps  # one kernel per step: the fused small-image kernel
    counters = load_counters(cfg)
    traffic = {k: v.get("dram_bytes") for k, v in counters.items()}
    if fused:
        # the whole step is one launch; its algorithmic bytes are the hybrid's 4 B/px
        ach = 4 * px_total / (ms_step * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": "hybrid_small_kernel (AMF + W1 fused)", "achieved": round(ach, 1),
                    "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                    "traffic": traffic.get("hybrid_small_kernel"), "peak_source": hbm_src,
                    "algorithmic_bytes_per_launch": 4 * px_total,
                    "step_achieved": round(ach, 1), "step_frac": round(ach / hbm, 4),
                    "kernel_ms": dict(kern, fused_ms=round(ms_step, 4))}
    elif kern:
        t_amf = kern["amf_ms"]
        t_w = kern["wiener_ms"] or 0.0
        dominant = "amf" if t_amf >= t_w else "wiener"
        if dominant == "amf":
            nbytes = 2 * px_total  # read g + write f, 1 B/px each
            ach = nbytes / (t_amf * 1e-3) / 1e9
            tr = traffic.get("amf")
        else:
            nbytes = 3 * px_total  # stats reads f, gain reads f + writes y
            ach = nbytes / (t_w * 1e-3) / 1e9
            tr = traffic.get("wiener")
        roofline = {"bound": "hbm", "kernel": dominant, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(ach / hbm, 4), "traffic": tr, "peak_source": hbm_src,
                    "algorithmic_bytes_per_launch": nbytes,
                    "step_achieved": round(4 * px_total / (ms_step * 1e-3) / 1e9, 1),
                    "step_frac": round(4 * px_total / (ms_step * 1e-3) / 1e9 / hbm, 4),
                    "kernel_ms": kern}
    # instruction-issue roofline (the north_star's second binding roofline: integer issue rate)
    issue = None
    sm_mhz = clk.report().get("sm_mhz")
    if fused:
        issue = issue_roofline("hybrid_small_kernel", counters, ms_step, sm_mhz)
    elif kern:
        issue = issue_roofline("amf", counters, kern["amf_ms"], sm_mhz)
        w_issue = issue_roofline("wiener", counters, kern.get("wiener_ms"), sm_mhz)
        if issue and w_issue:
            issue["wiener"] = {k: w_issue[k] for k in ("achieved", "frac")}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference(cfg, c, os.cpu_count() or 1, args.cpu_seconds)
        except Exception as e:  # the baseline is reported, never required
            cpu = {"unavailable": str(e)}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "MPix/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
        "scaling": "weak" if slices > 1 else "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload(cfg, c, world, not args.shared_gpu), "clocks": clk.report(), "e2e": e2e, "gpu_launches": int(launches), "issue_roofline": issue,
        "roofline": roofline, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="do not declare the GPU exclusive (hyb_set_exclusive): cooperative fused launches")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    from paper_2005_05371_b200 import CONFIGS
    c = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, args.config, c)
    return run_gpu(args, args.config, c)


if __name__ == "__main__":
    sys.exit(main())
