#!/usr/bin/env python3
"""Benchmark of the hybrid AMF + W1 Wiener hot path (BASELINE.json metric) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

A step is one pass of the hot path over one batch of synthetic input: one phantom image of the
chosen BASELINE.json config, or for config 3 the 512-slice stack.  The default workload is config 4
(16384^2, S&P 0.5, Smax 11, Wiener 7x7): the largest configuration that fits one GPU, on which the
headline is quoted; the other configs are parity-test cases and `--config` lines.

* ``value``: whole-job MPix/s with inputs resident in HBM (inputs larger than L2, or a rotating set
  of buffers > 3x L2, so every step reads cold data).
* ``e2e``: the same metric through the C ABI with pinned HOST buffers (H2D copy, kernels, D2H copy
  inside the timed region; at N > 1 each rank scatters its strip in and gathers its core rows out).
* N > 1: one process per GPU over NCCL -- strips with halo exchange + one int64 all-reduce (strip
  configs), or slice shards (config 3); both are strong scaling (the total work is fixed).  Run as
  ``python bench.py --gpus N`` (the script re-launches itself under torch.distributed.run) or under
  torchrun directly.
* ``--impl reference``: the reference's own CPU AMF (adaptive_median_parallel, compiled from the
  reference sources into oracle/_ref) + the W1 oracle on all host threads, on a bounded sample of the
  same workload.  That arm never imports the product package (no libhybrid_cuda.so is mapped).
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPix/s for hybrid AMF+Wiener (uint8) at 1/2/4/8 B200; % of roofline"
L2_BYTES = 126 * 1024 * 1024
DEFAULT_CONFIG = 4


def load_configs():
    """BASELINE.json configs from paper_2005_05371_b200/configs.py, loaded by path so the reference
    arm does not import the product package (whose __init__ maps libhybrid_cuda.so)."""
    spec = importlib.util.spec_from_file_location("_hyb_configs",
                                                  os.path.join(ROOT, "paper_2005_05371_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.CONFIGS


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


# min/max lane operations per pixel of the zmin / zmed / zmax selection for a k x k window (SURVEY.md 8(d)
# algorithmic work): k = 3 as the k = 3 kernel formulates it (10 column sorts reused by 3 outputs each +
# 8 three-input min/max per u16x2 output pair word, 168 ops per 16 pixels = 10.5 word ops = 21 lane ops
# per pixel); k >= 5: the pruned Batcher networks of tools/gen_networks.py, 2 ops per compare-exchange + 1
# per one-sided op (k = 5: 96 CE + 22, 7: 281 + 46, 9: 641 + 78, 11: 1030 + 118, 13: 1856 + 166,
# 15: 2546 + 222).
AMF_OPS = {3: 21, 5: 214, 7: 608, 9: 1360, 11: 2178, 13: 3878, 15: 5314}


def int_peak():
    """Measured VIMNMX.U16x2 throughput (tools/int_peak.cu on a B200, committed as profiles/int_peak.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "int_peak.json")) as f:
            return json.load(f)
    except Exception:
        return None


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

    def poll_until(self, event):
        """Sample synchronously until `event` (recorded after the timed launches) completes: the GPU is
        busy with the timed region the whole time, whatever the Python thread scheduling."""
        while not event.query():
            if self.nv:
                try:
                    self._sample()
                except Exception:
                    pass
            time.sleep(0.0005)

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
            time.sleep(0.001)

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


# ------------------------------------------------------------------------------------------------
# CPU baseline (reference arm and the cpu_baseline key): BASELINE.md section 4 / SURVEY.md 8(d)
# ------------------------------------------------------------------------------------------------

def host_info():
    model, ram = None, None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal:"):
                    ram = round(int(line.split()[1]) / 1024 / 1024, 1)
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model, "ram_gib": ram}


def cpu_sample(cfg, c, make_phantom):
    """A bounded sample of the config's workload for the CPU reference (about 10-30 s of CPU work
    for the whole protocol): single images -> a band of full-width rows from the middle of the
    phantom (filtered as its own image); config 3 -> the first 16 slices."""
    rows, cols = c["rows"], c["cols"]
    if c["slices"] > 1:
        n = min(16, c["slices"])
        imgs = [make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], s) for s in range(n)]
        return imgs, f"{n} of {c['slices']} {rows}x{cols} config-{cfg} slices (seeds 0..{n - 1})"
    img = make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], 0)
    band = {0: rows, 1: rows, 2: 1024, 4: 512}.get(cfg, rows)
    if band >= rows:
        return [img], f"the whole {rows}x{cols} config-{cfg} phantom (seed 0)"
    r0 = (rows - band) // 2
    return [img[r0:r0 + band].copy()], (f"rows [{r0}, {r0 + band}) x {cols} of the config-{cfg} phantom (seed 0), "
                                        f"filtered as one image")


def cpu_trial(oracle, imgs, c, threads):
    """One trial on the sample: the reference's adaptive_median_parallel (parts = workers = threads;
    compiled from the reference sources, oracle/_ref) + the W1 oracle on `threads` threads (the
    reference has no local Wiener).  Returns (seconds, pixels, kind)."""
    t, px = 0.0, 0
    kind = "reference" if oracle.ref_available() else "port"
    for img in imgs:
        if kind == "reference":
            _, ta, tw = oracle.ref_hybrid_baseline(img, c["smax"], c["win"], threads)
            t += ta + tw
        else:
            t0 = time.perf_counter()
            oracle.hybrid_threaded(img, c["smax"], c["win"], threads)
            t += time.perf_counter() - t0
        px += img.size
    return t, px, kind


def cpu_protocol(cfg, c):
    """cpu_baseline of the GPU arm: the paper's workers sweep (1/2/4/8 and all host
    threads, parts = workers), median of 3 trials each (proj/tools/hybridfilter.cpp:117), on a bounded
    sample; `value` is the all-threads point."""
    import oracle
    imgs, sample = cpu_sample(cfg, c, oracle.make_phantom)
    nproc = os.cpu_count() or 1
    sweep, kind, total = {}, None, 0.0
    for w in sorted({1, 2, 4, 8, nproc}):
        if w > nproc:
            continue
        ts = []
        for _ in range(3):
            t, px, kind = cpu_trial(oracle, imgs, c, w)
            ts.append(t)
            total += t
        sweep[str(w)] = round(px / statistics.median(ts) / 1e6, 3)
    return {"value": sweep[str(nproc)], "unit": "MPix/s", "cores": nproc, "kind": kind,
            "sample": sample + "; AMF = reference adaptive_median_parallel (parts = workers), Wiener = W1 oracle "
                               "(the reference has no local Wiener); median of 3 trials per worker count",
            "workers_sweep_mpix_s": sweep, "trials": 3, "cpu_seconds": round(total, 2), "host": host_info()}


def run_reference(args, cfg, c):
    """The reference arm: the reference's own CPU path on all host threads, each step one trial on a
    bounded sample of the workload.  Under torchrun only rank 0 works."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    threads = os.cpu_count() or 1
    imgs, sample = cpu_sample(cfg, c, oracle.make_phantom)
    per_step, kind = [], None
    for i in range(args.warmup + args.steps):
        t, px, kind = cpu_trial(oracle, imgs, c, threads)
        if i >= args.warmup:
            per_step.append((t, px))
    t_all = sum(t for t, _ in per_step)
    px_all = sum(px for _, px in per_step)
    value = px_all / t_all / 1e6
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "MPix/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_all / len(per_step) * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload(cfg, c, 1),
        "cpu_baseline": {"value": round(value, 3), "unit": "MPix/s", "cores": threads, "kind": kind,
                         "sample": sample + "; reference adaptive_median_parallel (parts = workers = all host "
                                            "threads) + W1 oracle on the same threads", "host": host_info()},
        "e2e": {"value": round(value, 3), "unit": "MPix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload(cfg, c, n, exclusive=True, nbuf=None):
    slices = c["slices"]
    d = {"workload": f"config{cfg}: {c['rows']}x{c['cols']} uint8 phantom"
            + (f" x {slices} slices" if slices > 1 else "")
            + f", {c['ellipses']} ellipses, sigma {c['sigma']}, S&P {c['density']}, AMF Smax {c['smax']}, "
              f"Wiener {c['win']}x{c['win']}",
            "pixels_per_step": c["rows"] * c["cols"] * slices,
            "partition": (f"{n} slice shards" if slices > 1 else f"{n} horizontal strips (halo exchange + one "
                          "int64 all-reduce per step)") if n > 1 else "1 GPU",
            }
    if nbuf is not None:  # GPU arm
        d["l2"] = (f"inputs larger than L2 ({c['rows'] * c['cols'] * slices / n / 2**20:.0f} MiB per rank per step "
                   f"> 126 MiB)" if nbuf == 1 else
                   f"{nbuf} rotating input/output buffers > 3x L2 (cold reads every step)")
        d["device_mode"] = ("exclusive (hyb_set_exclusive: plain persistent launches)" if exclusive
                            else "shared (cooperative launches)")
    return d


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------

def run_gpu(args, cfg, c):
    import numpy as np
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
    # the API default (cooperative launches of the fused small-image kernel) unless --exclusive declares the GPU
    # dedicated; configs 2-4 never take the fused kernel, so the mode only matters for configs 0 / 1
    ctx.set_exclusive(args.exclusive)
    lib = capi.lib

    rows, cols, slices = c["rows"], c["cols"], c["slices"]
    smax, win = c["smax"], c["win"]
    hbm, hbm_src = peaks()

    # ---------------- inputs (host phantom -> HBM) ----------------
    plan = None
    if slices > 1:
        my = [s for s in range(slices) if s % world == rank]
        host = torch.from_numpy(np.stack(
            [capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], s) for s in my]))
    else:
        img = torch.from_numpy(capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], 0))
        if world > 1:
            plan = StripPlan(rows, cols, smax, win, world, rank)
            host = img[plan.g_slice()].contiguous()
        else:
            host = img
    unit_bytes = host.numel()
    nbuf = max(1, math.ceil(3 * L2_BYTES / (2 * unit_bytes))) if unit_bytes <= L2_BYTES else 1
    g_bufs = [host.to(dev) for _ in range(nbuf)]
    if plan is not None:
        y_bufs = [torch.empty((plan.core, cols), dtype=torch.uint8, device=dev) for _ in g_bufs]
        backend = CudaStripBackend(ctx)
        f_strip = torch.empty((plan.f_rows, cols), dtype=torch.uint8, device=dev)
        w_dev = torch.zeros(1, dtype=torch.int64, device=dev)
    else:
        y_bufs = [torch.empty_like(g) for g in g_bufs]

    def step(i):
        g, y = g_bufs[i % nbuf], y_bufs[i % nbuf]
        if slices > 1:
            capi.check(lib.hyb_hybrid_batch_u8(ctx.ptr, g.data_ptr(), cols, rows * cols, g.shape[0], rows, cols,
                                               smax, win, y.data_ptr(), cols, rows * cols, None), ctx.ptr)
        elif plan is None:
            capi.check(lib.hyb_hybrid_u8(ctx.ptr, g.data_ptr(), cols, rows, cols, smax, win, 1, y.data_ptr(), cols,
                                         None), ctx.ptr)
        else:
            hybrid_strip_step(backend, plan, g, f_strip, y, w_dev)

    def timed(fn, k, sampler=None):
        """k calls of fn between a barrier + synchronize on both sides; CUDA events on the launch
        stream; the max over ranks.  `sampler` polls the clocks until the last launch completes."""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(k):
            fn(i)
        e1.record(stream)
        if sampler is not None:
            sampler.poll_until(e1)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # untimed warm-up: W steps, and at least two passes over the rotating buffers (the library
    # captures a CUDA graph per buffer pair on its second use and replays it afterwards)
    warm = max(args.warmup, 2 * nbuf)
    for i in range(warm):
        step(i)
    torch.cuda.synchronize()
    l0 = ctx.launches()
    with ClockSampler(local) as clk:
        ms = timed(step, args.steps, clk)
    launches = ctx.launches() - l0
    px_total = rows * cols * slices
    ms_step = ms / args.steps
    value = px_total / (ms_step * 1e-3) / 1e6

    # ---------------- per-stage breakdown (same inputs, CUDA events on the launch stream) --------
    # rank-local: this rank's image / strip / slice shard, no exchange or all-reduce
    g0 = g_bufs[0]
    nsl = g0.shape[0] if slices > 1 else 1
    a_rows = plan.g_rows if plan is not None else rows
    o_rows = (plan.f_rows if plan is not None else rows)
    rb = (plan.hA - plan.fa) if plan is not None else 0
    f_scr = [torch.empty((nsl, o_rows, cols) if slices > 1 else (o_rows, cols), dtype=torch.uint8, device=dev)
             for _ in range(nbuf)]
    px_local = a_rows * cols * nsl if slices > 1 else o_rows * cols

    def amf_only(i):
        g, f = g_bufs[i % nbuf], f_scr[i % nbuf]
        if slices > 1:
            capi.check(lib.hyb_amf_batch_u8(ctx.ptr, g.data_ptr(), cols, rows * cols, nsl, rows, cols, smax,
                                            f.data_ptr(), cols, rows * cols), ctx.ptr)
        else:
            capi.check(lib.hyb_amf_u8(ctx.ptr, g.data_ptr(), cols, a_rows, cols, rb, rb + o_rows, smax,
                                      f.data_ptr(), cols, None, cols), ctx.ptr)

    w_dev1 = torch.zeros(max(nsl, 1), dtype=torch.int64, device=dev)
    w_rows = plan.core if plan is not None else rows
    w_b = plan.fa if plan is not None else 0

    def wiener_only(i):
        f, y = f_scr[i % nbuf], y_bufs[i % nbuf]  # single images / strips only
        capi.check(lib.hyb_wiener_stats_u8(ctx.ptr, f.data_ptr(), cols, o_rows, cols, w_b, w_b + w_rows, win,
                                           w_dev1.data_ptr()), ctx.ptr)
        capi.check(lib.hyb_wiener_gain_u8(ctx.ptr, f.data_ptr(), cols, o_rows, cols, w_b, w_b + w_rows, win,
                                          w_dev1.data_ptr(), rows * cols, y.data_ptr(), cols), ctx.ptr)

    # stage timings below are rank-local (this rank's work alone, no max over ranks)

    def timed_local(fn, k):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(k):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for i in range(3):
        amf_only(i)
    k_stage = max(args.steps, 10)
    t_amf = timed_local(amf_only, k_stage) / k_stage
    t_w = None
    if slices == 1:
        for i in range(3):
            wiener_only(i)
        t_w = timed_local(wiener_only, k_stage) / k_stage
    kern = {"amf_ms": round(t_amf, 4), "wiener_ms": round(t_w, 4) if t_w else None}

    # algorithmic work of the AMF: for every window size k a pixel reaches, the min/max lane
    # operations of a selection network giving zmin / zmed / zmax (AMF_OPS), summed from this rank's
    # finalized_at histogram (the kernels' finalized_at is bit-exact vs the oracle, tests/test_gpu_parity.py;
    # unresolved pixels (0) reached every level).  Element visits sum_k reach(k) k^2 are kept beside it.
    visits = ops = None
    if slices == 1:
        fin = torch.empty((o_rows, cols), dtype=torch.uint8, device=dev)
        capi.check(lib.hyb_amf_u8(ctx.ptr, g0.data_ptr(), cols, a_rows, cols, rb, rb + o_rows, smax,
                                  f_scr[0].data_ptr(), cols, fin.data_ptr(), cols), ctx.ptr)
        torch.cuda.synchronize()
        hist = torch.bincount(fin.flatten().long(), minlength=256).cpu().numpy()
        visits = ops = 0
        for k in range(3, smax + 1, 2):
            reach = int(hist[0]) + int(hist[k:].sum())  # finalised at >= k, or never
            visits += reach * k * k
            ops = ops + reach * AMF_OPS[k] if (ops is not None and k in AMF_OPS) else None
        del fin

    # ---------------- e2e through the C ABI with pinned host buffers ----------------
    h_in = host.pin_memory()
    out_rows = plan.core if plan is not None else None
    h_out = (torch.empty((out_rows, cols), dtype=torch.uint8).pin_memory() if plan is not None
             else torch.empty_like(h_in).pin_memory())
    if plan is not None:
        g_e2e = torch.empty_like(g_bufs[0])
        y_e2e = torch.empty((plan.core, cols), dtype=torch.uint8, device=dev)

    def e2e_step(i):
        if slices > 1:
            capi.check(lib.hyb_hybrid_batch_u8(ctx.ptr, h_in.data_ptr(), cols, rows * cols, h_in.shape[0], rows,
                                               cols, smax, win, h_out.data_ptr(), cols, rows * cols, None),
                       ctx.ptr)
        elif plan is None:
            capi.check(lib.hyb_hybrid_u8(ctx.ptr, h_in.data_ptr(), cols, rows, cols, smax, win, 1,
                                         h_out.data_ptr(), cols, None), ctx.ptr)
        else:
            # scatter: this rank's strip (core + halo rows) from the host; gather: its core rows back
            g_e2e.copy_(h_in, non_blocking=True)
            hybrid_strip_step(backend, plan, g_e2e, f_strip, y_e2e, w_dev, exchange=False)
            h_out.copy_(y_e2e, non_blocking=True)

    for i in range(max(2, args.warmup)):
        e2e_step(i)
    torch.cuda.synchronize()
    k_e2e = max(1, args.steps)  # the same K as the device-resident loop
    t0 = time.perf_counter()
    ms_e2e = timed(e2e_step, k_e2e)
    wall = (time.perf_counter() - t0) / k_e2e
    e2e_sync = {"value": round(px_total / (ms_e2e / k_e2e * 1e-3) / 1e6, 3), "ms_per_step": round(ms_e2e / k_e2e, 4),
                "wall_ms_per_step": round(wall * 1e3, 4)}
    e2e = dict(e2e_sync, unit="MPix/s", h2d_bytes_per_step=int(h_in.numel()) * world,
               d2h_bytes_per_step=int(h_out.numel()) * world, mode="synchronous calls")
    if plan is None and slices == 1:
        # a stream of images through the asynchronous host API (hyb_set_async): each call still uploads its
        # input from pinned host memory and downloads its result, but call i + 1's upload overlaps call i's
        # download; the timed region ends after hyb_synchronize (every result back in host memory)
        h_outs = [h_out, torch.empty_like(h_out).pin_memory()]
        ctx.set_async(True)

        def e2e_async(i):
            capi.check(lib.hyb_hybrid_u8(ctx.ptr, h_in.data_ptr(), cols, rows, cols, smax, win, 1,
                                         h_outs[i % 2].data_ptr(), cols, None), ctx.ptr)

        for i in range(max(2, args.warmup)):
            e2e_async(i)
        ctx.synchronize()
        torch.cuda.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ea.record(stream)
        for i in range(k_e2e):
            e2e_async(i)
        ctx.synchronize()  # joins the copy streams into `stream`, waits for everything
        eb.record(stream)
        eb.synchronize()
        wall_a = (time.perf_counter() - t0) / k_e2e
        ms_a = ea.elapsed_time(eb) / k_e2e
        ctx.set_async(False)
        e2e = {"value": round(px_total / (ms_a * 1e-3) / 1e6, 3), "unit": "MPix/s",
               "h2d_bytes_per_step": int(h_in.numel()), "d2h_bytes_per_step": int(h_out.numel()),
               "ms_per_step": round(ms_a, 4), "wall_ms_per_step": round(wall_a * 1e3, 4),
               "mode": "asynchronous host API (hyb_set_async): K images back to back, upload of image i+1 "
                       "overlapping the download of image i; timed to hyb_synchronize",
               "synchronous": e2e_sync}
    if plan is not None:
        e2e["note"] = ("per rank: H2D of its strip (core + halo rows, the halo rows come from the host copy "
                       "instead of the exchange), strip step, D2H of its core rows; max over ranks")

    # rank 0 reports; gather the per-rank stage timings for the line
    stage = torch.tensor([t_amf, t_w or 0.0, float(visits or 0), float(px_local)], device=dev, dtype=torch.float64)
    if world > 1:
        allst = [torch.zeros_like(stage) for _ in range(world)]
        dist.all_gather(allst, stage)
        allst = [s.cpu().tolist() for s in allst]
    else:
        allst = [stage.cpu().tolist()]
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---------------- roofline of the dominant stage ----------------
    counters = load_counters(cfg)
    traffic = {k: v.get("dram_bytes") for k, v in counters.items()}
    fused = world == 1 and launches == args.steps  # one kernel per step: the fused small-image kernel
    sm_mhz = clk.report().get("sm_mhz")
    if fused:
        # the whole step is one launch; its algorithmic bytes are the hybrid's 4 B/px
        ach = 4 * px_total / (ms_step * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": "hybrid_small_kernel (AMF + W1 fused)", "achieved": round(ach, 1),
                    "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                    "traffic": traffic.get("hybrid_small_kernel"), "peak_source": hbm_src,
                    "algorithmic_bytes_per_launch": 4 * px_total,
                    "kernel_ms": dict(kern, fused_ms=round(ms_step, 4))}
        issue = issue_roofline("hybrid_small_kernel", counters, ms_step, sm_mhz)
    else:
        dominant = "amf" if t_amf >= (t_w or 0.0) else "wiener"
        if dominant == "amf":
            nbytes = 2 * px_local  # read g + write f, 1 B/px each
            ach = nbytes / (t_amf * 1e-3) / 1e9
        else:
            nbytes = 3 * px_local  # statistics read f; gain reads f, writes y
            ach = nbytes / (t_w * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": dominant + (" (amf_k3_kernel + amf_grow_kernel)" if dominant == "amf"
                                                          else " (w1 statistics + gain)"),
                    "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                    "traffic": traffic.get(dominant) if world == 1 else None, "peak_source": hbm_src,
                    "algorithmic_bytes_per_launch": nbytes,
                    "step_achieved": round(4 * px_total / world / (ms_step * 1e-3) / 1e9, 1),
                    "step_frac": round(4 * px_total / world / (ms_step * 1e-3) / 1e9 / hbm, 4),
                    "kernel_ms": kern}
        if world > 1:
            roofline["per_gpu"] = "rank 0's strip stage timed alone (no exchange / all-reduce); step_* = whole-job " \
                                  "4 B/px over all ranks / N"
        issue = issue_roofline("amf", counters, t_amf, sm_mhz) if world == 1 else None
        if issue:
            w_issue = issue_roofline("wiener", counters, t_w, sm_mhz)
            if w_issue:
                issue["wiener"] = {k: w_issue[k] for k in ("achieved", "frac")}

    # integer roofline of the AMF: algorithmic min/max lane operations / s vs the measured VIMNMX.U16x2
    # lane rate (two 16-bit lanes per instruction)
    int_roof = None
    ip = int_peak()
    if ops and ip:
        ach = ops / (t_amf * 1e-3) / 1e9
        pk = ip["elem_per_s"] / 1e9
        int_roof = {"bound": "integer ALU (VIMNMX.U16x2 lane min/max)", "kernel": "amf (k3 + growth)",
                    "achieved": round(ach, 1), "peak": round(pk, 1), "unit": "G min/max lane-ops/s",
                    "frac": round(ach / pk, 4),
                    "work_per_px": round(ops / px_local, 3),
                    "work": "sum_k reach(k) * ops(k): min/max lane operations of a zmin/zmed/zmax selection "
                            "network for every window size the pixel reaches (k = 3: shared 3-tall column "
                            "sorts, 21 ops/px; k >= 5: the pruned Batcher networks of tools/gen_networks.py, "
                            "214 / 608 / 1360 / 2178 ops at k = 5 / 7 / 9 / 11), reach(k) from the "
                            "finalized_at histogram of this input; a 3-input min/max counts as 2 ops",
                    "element_visits_per_px": round(visits / px_local, 3),
                    "peak_source": "profiles/int_peak.json (tools/int_peak.cu, " + ip.get("how", "") + ")"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_protocol(cfg, c)
        except Exception as e:  # the baseline is reported, never required
            cpu = {"unavailable": str(e)}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "MPix/s", "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload(cfg, c, world, args.exclusive, nbuf), "clocks": clk.report(), "e2e": e2e,
        "gpu_launches": int(launches), "roofline": roofline, "int_roofline": int_roof, "issue_roofline": issue,
        "cpu_baseline": cpu,
    }
    if warm != args.warmup:
        line["warmup_requested"] = args.warmup
    if world > 1:
        line["per_rank_stage_ms"] = [{"amf_ms": round(s[0], 4), "wiener_ms": round(s[1], 4)} for s in allst]
        line["nccl_debug"] = os.environ.get("NCCL_DEBUG")
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------------------------------
# launcher
# ------------------------------------------------------------------------------------------------

def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args):
    """`python bench.py --gpus N` without torchrun: run the same command under torch.distributed.run,
    one process per GPU on this node, rendezvous on 127.0.0.1."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the communicator lines show nranks / the transport
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def check_launch(args, cfg, c):
    """--check-launch (CPU, gloo): the launcher and the rank plumbing of the N > 1 path without a GPU --
    every rank builds its strip plan, fills its core rows from a deterministic pattern, exchanges halos
    (the same exchange_halos the NCCL path runs), all-reduces a checksum and the max of its step time;
    rank 0 prints one JSON line.  Used by tests/test_bench_launcher.py."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2005_05371_b200.partition import StripPlan, exchange_halos

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist.init_process_group("gloo")
    rows, cols = 256, 64
    img = (np.arange(rows * cols, dtype=np.int64).reshape(rows, cols) * 2654435761 % 251).astype(np.uint8)
    plan = StripPlan(rows, cols, c["smax"], c["win"], world, rank)
    g = torch.zeros((plan.g_rows, cols), dtype=torch.uint8)
    g[plan.hA:plan.hA + plan.core] = torch.from_numpy(img[plan.core_slice()])
    t0 = time.perf_counter()
    exchange_halos(plan, g)
    ok = torch.tensor([int((g.numpy() == img[plan.g_slice()]).all())], dtype=torch.int64)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"check": "launch", "n_gpus": world, "world_size": world, "halos_ok": bool(ok.item()),
                          "ms_max_over_ranks": round(float(ms.item()), 3),
                          "master_addr": os.environ.get("MASTER_ADDR")}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok.item() else 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--check-launch", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--exclusive", action="store_true",
                    help="declare the GPU dedicated (hyb_set_exclusive): plain instead of cooperative launches of "
                         "the fused small-image kernel (configs 0 / 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.gpus > 1 and not args.check_launch:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    configs = load_configs()
    c = configs[args.config]
    if args.check_launch:
        return check_launch(args, args.config, c)
    if args.impl == "reference":
        return run_reference(args, args.config, c)
    return run_gpu(args, args.config, c)


if __name__ == "__main__":
    sys.exit(main())
