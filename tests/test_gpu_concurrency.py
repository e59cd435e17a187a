"""Races between concurrent approximations (compute-sanitizer is closed on this GPU pool, so the
evidence is behavioural): two native contexts on two streams, each replaying its approximation
as a CUDA graph while the other runs (the bench's two-in-flight mode), and a batched call whose
lanes overlap, must reproduce the bits of a solitary run every time, on both engines."""
import pytest
import torch

from paper_2402_19147_b200 import _native
from paper_2402_19147_b200.cur import DeviceApprox, DeviceBatch
from paper_2402_19147_b200.quat import to_device
from helpers import lowrank

pytestmark = pytest.mark.gpu


def snapshot(o):
    return [t.clone() for t in (o.J, o.I, o.C, o.U, o.R, o.err4)]


@pytest.mark.parametrize("mode", [1, 2])
def test_two_contexts_in_flight_bitwise(mode):
    m, n, c, r = 1200, 1100, 64, 60
    devs = [_native.Device(0), _native.Device(0)]
    xs = [to_device(lowrank(m, n, 12, seed=70 + k, noise=1e-3), devs[k]) for k in range(2)]
    outs = [DeviceApprox(m, n, c, r, devs[k]) for k in range(2)]
    streams = [torch.cuda.Stream(0), torch.cuda.Stream(0)]
    for d in devs:
        d.call("qcur_set_gemm_mode", mode)
    ref = []
    for k in range(2):  # solitary runs
        with torch.cuda.stream(streams[k]):
            outs[k].run(xs[k], "length", 9 + k)
        torch.cuda.synchronize()
        outs[k].check()
        ref.append(snapshot(outs[k]))
    for rep in range(10):  # both in flight, graph replays interleaved on two streams
        for k in range(2):
            with torch.cuda.stream(streams[k]):
                outs[k].run(xs[k], "length", 9 + k, graph=True)
        torch.cuda.synchronize()
        for k in range(2):
            outs[k].check()
            for a, b in zip(snapshot(outs[k]), ref[k]):
                assert torch.equal(a, b), (rep, k)


def test_batched_lanes_repeatable():
    dev = _native.device()
    B, m, n, c, r = 8, 400, 380, 32, 30
    xs = [to_device(lowrank(m, n, 8, seed=200 + b, noise=1e-3), dev) for b in range(B)]
    bt = DeviceBatch(B, m, n, c, r, dev, lanes=8)
    bt.run(xs, "length", list(range(B)))
    bt.check()
    ref = [t.clone() for t in (bt.J, bt.I, bt.U, bt.err4)]
    for _ in range(10):
        bt.run(xs, "length", list(range(B)), graph=True)
        torch.cuda.synchronize()
        bt.check()
        for a, b in zip((bt.J, bt.I, bt.U, bt.err4), ref):
            assert torch.equal(a, b)
