"""Multi-GPU strip partitioner: one process per GPU over torch.distributed (NCCL on B200).

Mirrors adaptive_median_parallel's band decomposition (reference proj/src/parallel.cpp:27-70,
band heights proj/src/tiling.cpp:23-32) with one band per rank, the paper's workers = parts case.
Per step each rank

  1. refreshes the halo rows of its g strip from its neighbours (rank-1 / rank+1 send their
     boundary CORE rows; one send/recv pair per neighbour, NCCL P2P over NVLink),
  2. runs the AMF on its core rows plus rW rows on each side (redundant rows, so the Wiener
     stats of its core rows need no second exchange; halo depth rA + rW),
  3. adds its core rows' W = sum V into a device int64 and all-reduces it (ONE collective of
     8 bytes per image -- exact integers, so the result is identical to 1 GPU),
  4. applies the gain to its core rows.

The compute is injected (``StripBackend``) so the exchange / reduction logic runs under gloo on
the CPU in tests with the oracle as the backend; the product backend is ``CudaStripBackend``.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .denoise import split_bands


@dataclass
class StripPlan:
    rows: int
    cols: int
    smax: int
    win: int
    world: int
    rank: int

    def __post_init__(self):
        self.rA = (self.smax - 1) // 2
        self.rW = (self.win - 1) // 2
        self.h = self.rA + self.rW
        self.bands = split_bands(self.rows, self.world, self.h)
        b = self.bands[self.rank]
        self.start, self.core = b.core_start, b.core_rows
        self.hA, self.hB = b.halo_above, b.halo_below
        self.fa = min(self.rW, self.start)
        self.fb = min(self.rW, self.rows - self.start - self.core)
        for nb in self.bands:
            if nb.core_rows < self.h and self.world > 1:
                raise ValueError(f"strip of {nb.core_rows} rows is thinner than the halo {self.h}; "
                                 "use fewer ranks for this image")

    @property
    def g_rows(self):  # rows of the local g buffer (halo + core + halo)
        return self.hA + self.core + self.hB

    @property
    def f_rows(self):
        return self.fa + self.core + self.fb

    def core_slice(self):
        return slice(self.start, self.start + self.core)

    def g_slice(self):
        return slice(self.start - self.hA, self.start + self.core + self.hB)


def exchange_halos(plan: StripPlan, g_strip: torch.Tensor, group=None) -> None:
    """Fill g_strip's halo rows from the neighbours' core rows (in place)."""
    if plan.world == 1:
        return
    ops = []
    up, down = plan.rank - 1, plan.rank + 1
    core0 = plan.hA
    core1 = plan.hA + plan.core
    if plan.rank > 0:
        # my top hA halo rows are the last hA core rows of rank-1; it needs my first rows
        ops.append(dist.P2POp(dist.irecv, g_strip[0:plan.hA], up, group))
        n_up = plan.bands[up].halo_below
        ops.append(dist.P2POp(dist.isend, g_strip[core0:core0 + n_up].contiguous(), up, group))
    if plan.rank < plan.world - 1:
        ops.append(dist.P2POp(dist.irecv, g_strip[core1:core1 + plan.hB], down, group))
        nb = plan.bands[down]
        n_down = nb.halo_above
        ops.append(dist.P2POp(dist.isend, g_strip[core1 - n_down:core1].contiguous(), down, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


class StripBackend:
    """Per-strip compute used by ``hybrid_strip_step``."""

    def amf(self, g_strip, plan: StripPlan, f_strip):  # f rows = g rows [hA-fa, hA+core+fb)
        raise NotImplementedError

    def stats(self, f_strip, plan: StripPlan, w):  # w += sum V over f rows [fa, fa+core)
        raise NotImplementedError

    def gain(self, f_strip, plan: StripPlan, w, y_core):
        raise NotImplementedError


def hybrid_strip_step(backend: StripBackend, plan: StripPlan, g_strip, f_strip, y_core, w, group=None,
                      exchange: bool = True):
    """One hybrid pass over this rank's strip; w is a 1-element int64 tensor (device for NCCL)."""
    if exchange:
        exchange_halos(plan, g_strip, group)
    backend.amf(g_strip, plan, f_strip)
    w.zero_()
    backend.stats(f_strip, plan, w)
    if plan.world > 1:
        dist.all_reduce(w, op=dist.ReduceOp.SUM, group=group)
    backend.gain(f_strip, plan, w, y_core)


class CudaStripBackend(StripBackend):
    """The product: libhybrid_cuda kernels on this rank's GPU, no host synchronisation."""

    def __init__(self, ctx):
        from . import capi
        self.capi = capi
        self.ctx = ctx

    def amf(self, g_strip, plan, f_strip):
        c = self.capi
        c.check(c.lib.hyb_amf_u8(self.ctx.ptr, g_strip.data_ptr(), g_strip.stride(0), plan.g_rows, plan.cols,
                                 plan.hA - plan.fa, plan.hA + plan.core + plan.fb, plan.smax,
                                 f_strip.data_ptr(), f_strip.stride(0), None, plan.cols), self.ctx.ptr)

    def stats(self, f_strip, plan, w):
        c = self.capi
        c.check(c.lib.hyb_wiener_stats_u8(self.ctx.ptr, f_strip.data_ptr(), f_strip.stride(0), plan.f_rows,
                                          plan.cols, plan.fa, plan.fa + plan.core, plan.win, w.data_ptr()),
                self.ctx.ptr)

    def gain(self, f_strip, plan, w, y_core):
        c = self.capi
        c.check(c.lib.hyb_wiener_gain_u8(self.ctx.ptr, f_strip.data_ptr(), f_strip.stride(0), plan.f_rows,
                                         plan.cols, plan.fa, plan.fa + plan.core, plan.win, w.data_ptr(),
                                         plan.rows * plan.cols, y_core.data_ptr(), y_core.stride(0)),
                self.ctx.ptr)
