"""CPU, world_size 2 and 3 over gloo: the one-process-per-GPU strip partitioner (halo exchange by
send/recv, one all-reduce of the exact int64 noise sum) with the C oracle standing in for the
kernels.  The stitched result must equal the single-image oracle bit for bit -- the multi-GPU
analogue of the reference's partition-invariance tests (proj/tests/test_parallel.cpp:54-76)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2005_05371_b200.partition import StripBackend, StripPlan, hybrid_strip_step


class OracleBackend(StripBackend):
    def amf(self, g_strip, plan, f_strip):
        f_strip.copy_(torch.from_numpy(oracle.amf(g_strip.numpy(), plan.smax, plan.hA - plan.fa,
                                                  plan.hA + plan.core + plan.fb)))

    def stats(self, f_strip, plan, w):
        w += oracle.wiener_stats(f_strip.numpy(), plan.win, plan.fa, plan.fa + plan.core)

    def gain(self, f_strip, plan, w, y_core):
        y_core.copy_(torch.from_numpy(oracle.wiener_gain(f_strip.numpy(), plan.win, int(w.item()),
                                                         plan.rows * plan.cols, plan.fa, plan.fa + plan.core)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, img, smax, win, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows, cols = img.shape
    plan = StripPlan(rows, cols, smax, win, world, rank)
    g = torch.zeros((plan.g_rows, cols), dtype=torch.uint8)
    g[plan.hA:plan.hA + plan.core] = torch.from_numpy(img[plan.core_slice()])  # halos arrive by exchange
    f = torch.empty((plan.f_rows, cols), dtype=torch.uint8)
    y = torch.empty((plan.core, cols), dtype=torch.uint8)
    w = torch.zeros(1, dtype=torch.int64)
    hybrid_strip_step(OracleBackend(), plan, g, f, y, w)
    halo_ok = bool((g.numpy() == img[plan.g_slice()]).all())
    out_q.put((rank, plan.start, y.numpy().copy(), int(w.item()), halo_ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,smax,win", [(2, (61, 45), 7, 3), (3, (80, 33), 9, 5), (2, (50, 64), 11, 7)])
def test_strip_partition_matches_single_image(world, shape, smax, win):
    rng = np.random.default_rng(world * 100 + smax)
    img = rng.integers(0, 256, shape, dtype=np.uint8)
    img[rng.random(shape) < 0.15] = 0
    img[rng.random(shape) < 0.15] = 255
    ref_y, ref_w = oracle.hybrid(img, smax, win)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, img, smax, win, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = np.zeros_like(img)
    for rank, start, part, w, halo_ok in res:
        assert halo_ok, f"rank {rank} halo rows differ from the image"
        assert w == ref_w
        y[start:start + part.shape[0]] = part
    np.testing.assert_array_equal(y, ref_y)
