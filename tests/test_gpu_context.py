"""Context lifecycle on the GPU: cached CUDA graphs across scratch reallocation, per-context launch
counters, and the Python mirror's choice of context."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from paper_2005_05371_b200 import capi, denoise

pytestmark = pytest.mark.gpu


def _img(rows, cols, seed):
    return capi.make_phantom(rows, cols, 8, 12.0, 0.25, seed)


def _hybrid(ctx, g, y, smax=7, win=3, parts=1):
    rows, cols = g.shape
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, g.data_ptr(), cols, rows, cols, smax, win, parts, y.data_ptr(), cols,
                                      None), ctx.ptr)


def test_graph_replay_after_scratch_reallocation():
    """A graph captured over the context's scratch must not be replayed after a larger call (or a
    batch, or more strips) reallocated that scratch (replay over freed memory)."""
    ctx = capi.Context(0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    ctx.set_exclusive(True)
    with torch.cuda.stream(stream):
        ga = torch.from_numpy(_img(2100, 1900, 1)).cuda()  # separate-kernel path (> fused-kernel size)
        gb = torch.from_numpy(_img(4200, 3000, 2)).cuda()  # larger: f and the AMF workspace grow
        ya, yb = torch.empty_like(ga), torch.empty_like(gb)
        ref_a = oracle.hybrid_threaded(ga.cpu().numpy(), 7, 3)[0]
        ref_b = oracle.hybrid_threaded(gb.cpu().numpy(), 7, 3)[0]
        stack = torch.from_numpy(np.stack([_img(256, 256, s) for s in range(40)])).cuda()
        ys = torch.empty_like(stack)
        for it in range(3):  # plain run, capture, replay
            ya.zero_()
            _hybrid(ctx, ga, ya)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(ya.cpu().numpy(), ref_a, err_msg=f"a, call {it}")
        for it in range(3):
            _hybrid(ctx, gb, yb)  # reallocates the scratch the graph of `a` was captured over
            ya.zero_()
            _hybrid(ctx, ga, ya)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(ya.cpu().numpy(), ref_a, err_msg=f"a after b, round {it}")
            np.testing.assert_array_equal(yb.cpu().numpy(), ref_b, err_msg=f"b, round {it}")
            denoise.hybrid_denoise_batch(stack, 7, 3, ctx=ctx)  # batch scratch (noise sums per slice)
            _hybrid(ctx, ga, ya, parts=4)  # strip buffers
            ya.zero_()
            _hybrid(ctx, ga, ya)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(ya.cpu().numpy(), ref_a, err_msg=f"a after batch/strips, round {it}")
    ctx.close()


def test_launch_counters_are_per_context():
    a, b = capi.Context(0), capi.Context(0)
    g = torch.from_numpy(_img(600, 700, 3)).cuda()
    y = torch.empty_like(g)
    la, lb = a.launches(), b.launches()
    _hybrid(a, g, y)
    torch.cuda.synchronize()
    assert a.launches() > la
    assert b.launches() == lb
    a.close()
    b.close()


def test_mirror_uses_the_inputs_device_context():
    g = torch.from_numpy(_img(300, 300, 4)).cuda()
    res = denoise.hybrid_denoise(g, denoise.FilterConfig(smax=7, wiener_window=3))
    np.testing.assert_array_equal(res.image.cpu().numpy(), oracle.hybrid(g.cpu().numpy(), 7, 3)[0])
    # a context bound to another device than the tensor's is rejected (here: a fake device index)
    fake = capi.default_context(0)
    real_dev = fake.device
    try:
        fake.device = 1
        with pytest.raises(capi.InvalidArgument):
            denoise.hybrid_denoise(g, denoise.FilterConfig(smax=7, wiener_window=3), ctx=fake)
    finally:
        fake.device = real_dev


@pytest.mark.parametrize("shape", [(300, 420), (3000, 2900)])  # one-piece (fused kernel) and chunked pipelines
def test_async_host_calls_pipeline_bit_exact(shape):
    """hyb_set_async: calls on pinned host buffers return once enqueued; consecutive calls overlap (double-
    buffered staging); after synchronize() every output equals the oracle, and the context returns to
    synchronous behaviour."""
    ctx = capi.Context(0)
    ctx.set_exclusive(True)
    rows, cols = shape
    imgs = [torch.from_numpy(_img(rows, cols, 20 + i)).pin_memory() for i in range(5)]
    outs = [torch.empty((rows, cols), dtype=torch.uint8).pin_memory() for _ in range(5)]
    refs = [oracle.hybrid_threaded(g.numpy(), 9, 5)[0] for g in imgs]
    ctx.set_async(True)
    for rep in range(2):
        for o in outs:
            o.zero_()
        for g, o in zip(imgs, outs):
            capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, g.data_ptr(), cols, rows, cols, 9, 5, 1, o.data_ptr(), cols,
                                              None), ctx.ptr)
        ctx.synchronize()
        for i, (o, r) in enumerate(zip(outs, refs)):
            np.testing.assert_array_equal(o.numpy(), r, err_msg=f"rep {rep} image {i}")
    ctx.set_async(False)
    outs[0].zero_()
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, imgs[0].data_ptr(), cols, rows, cols, 9, 5, 1, outs[0].data_ptr(), cols,
                                      None), ctx.ptr)
    np.testing.assert_array_equal(outs[0].numpy(), refs[0])  # synchronous again: complete on return
    ctx.close()
