"""Throughput API: a stream of host matrices through the QMCUR path with the
host-to-device copy of matrix k+1 overlapped with the computation of matrix k.

The reference runs its approximations one after another on the CPU (the trial
loops of bench.py:243-352 and cli.py call make_plan + qmcur per matrix).  On the
B200 a cfg2 approximation takes ~8.8 ms of device time while moving its 512 MB
input over PCIe takes ~9.4 ms, so a one-at-a-time caller leaves either the link
or the SMs idle.  ``approx_stream`` keeps both busy: one native context uploads
(and interleaves) the next matrix on its own stream into a ping-pong device
buffer while a second context runs the whole approximation (K1..K9, qcur_approx)
on the current one; results (indices, U, the error statistics) come back with
small device-to-host copies.  The numbers are exactly those of
make_plan + qmcur + cur_relative_error on the same matrix and seed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, Iterator

import numpy as np

from . import _native
from .cur import _check_strategy, default_sample_counts
from .errors import ShapeError
from .quat import QMatrix, as_planes

__all__ = ["StreamResult", "approx_stream"]


_ctx_cache: dict = {}


def _stream_contexts(index: int):
    """(upload context, compute context, upload stream, compute stream) for a device,
    created once per process: each native context owns its workspace arena."""
    hit = _ctx_cache.get(index)
    if hit is None:
        torch = _native.device(index).torch
        hit = (_native.Device(index), _native.Device(index), torch.cuda.Stream(index), torch.cuda.Stream(index))
        _ctx_cache[index] = hit
    return hit


@dataclass(frozen=True)
class StreamResult:
    index: int
    row_indices: np.ndarray
    col_indices: np.ndarray
    u: QMatrix
    rel_err: float

    def factors(self, x):
        """C = X[:, J], R = X[I, :] on the host (the reference's take_cols / take_rows)."""
        planes = as_planes(x)
        c = QMatrix(*(p[:, self.col_indices] for p in planes))
        r = QMatrix(*(p[self.row_indices, :] for p in planes))
        return c, self.u, r


def approx_stream(matrices: Iterable, strategy: str, rank: int, seeds, num_rows: int | None = None,
                  num_cols: int | None = None) -> Iterator[StreamResult]:
    """Approximate every matrix of `matrices` (host QMatrix-like, all of one shape) with
    make_plan(x, strategy, rank, seed) + qmcur + relative error; seeds: one per matrix
    (iterable) or an int used for all.  Yields results in input order."""
    _check_strategy(strategy)
    torch = _native.device().torch
    up, comp, s_up, s_comp = _stream_contexts(torch.cuda.current_device())
    seed_iter = iter(seeds) if not isinstance(seeds, (int, np.integer)) else None
    shape = None
    slots = []
    pending = []  # (index, slot, done_event)
    code = _native.STRATEGY_CODES[strategy]

    def finish(item):
        idx, sl, ev = item
        ev.synchronize()
        comp.check(comp.lib.qcur_status_map(comp.handle, int(sl["st_h"][0])))  # this matrix's status
        e2, x2 = float(sl["err_h"][0]), float(sl["err_h"][1])
        u = QMatrix(*(np.array(sl["u_h"][:, :, k]) for k in range(4)))
        return StreamResult(index=idx, row_indices=np.array(sl["i_h"]), col_indices=np.array(sl["j_h"]), u=u,
                            rel_err=math.sqrt(e2) / math.sqrt(x2))

    for k, x in enumerate(matrices):
        planes = [np.ascontiguousarray(p, dtype=np.float64) for p in as_planes(x)]
        m, n = planes[0].shape
        if shape is None:
            shape = (m, n)
            d_rows, d_cols = default_sample_counts(rank, m, n)
            r = int(num_rows if num_rows is not None else d_rows)
            c = int(num_cols if num_cols is not None else d_cols)
            for _ in range(2):
                slots.append(dict(
                    x=comp.empty_q(m, n), J=comp.empty(c, dtype=torch.int64), I=comp.empty(r, dtype=torch.int64),
                    C=comp.empty_q(m, c), U=comp.empty_q(c, r), R=comp.empty_q(r, n), err=comp.empty(4),
                    u_h=torch.empty((c, r, 4), dtype=torch.float64, pin_memory=True).numpy(),
                    j_h=torch.empty(c, dtype=torch.int64, pin_memory=True).numpy(),
                    i_h=torch.empty(r, dtype=torch.int64, pin_memory=True).numpy(),
                    err_h=torch.empty(4, dtype=torch.float64, pin_memory=True).numpy(),
                    st_h=torch.empty(1, dtype=torch.int32, pin_memory=True).numpy(),
                    up_done=torch.cuda.Event(), used=torch.cuda.Event(), done=torch.cuda.Event()))
        elif (m, n) != shape:
            raise ShapeError(f"matrix {k} has shape {(m, n)}, the stream's is {shape}")
        seed = int(next(seed_iter)) if seed_iter is not None else int(seeds)
        sl = slots[k % 2]
        # at most one older matrix is in flight: the slot's previous user (k - 2) has been
        # yielded, so its host buffers are free and `used` orders the device side
        while len(pending) > 1:
            yield finish(pending.pop(0))
        with torch.cuda.stream(s_up):  # upload on its own stream once the slot's x is released
            s_up.wait_event(sl["used"])
            up.call("qcur_upload_planar", *(p.ctypes.data for p in planes), m, n, sl["x"].data_ptr())
            sl["up_done"].record(s_up)
        with torch.cuda.stream(s_comp):
            s_comp.wait_event(sl["up_done"])
            st = _native.state_from_seed(seed)
            comp.call("qcur_approx", sl["x"].data_ptr(), m, n, code, st.ctypes.data_as(_native._u64p), c, r,
                      sl["J"].data_ptr(), sl["I"].data_ptr(), sl["C"].data_ptr(), sl["U"].data_ptr(),
                      sl["R"].data_ptr(), 0.0, _native.CORE_CODES["projection"], sl["err"].data_ptr())
            sl["used"].record(s_comp)
            for dst, src in (("u_h", "U"), ("j_h", "J"), ("i_h", "I"), ("err_h", "err")):
                torch.from_numpy(sl[dst]).copy_(sl[src], non_blocking=True)
            comp.call("qcur_status_async", sl["st_h"].ctypes.data)
            sl["done"].record(s_comp)
        pending.append((k, sl, sl["done"]))
        if len(pending) > 1:  # the previous matrix finishes while this one uploads / runs
            yield finish(pending.pop(0))
    while pending:
        yield finish(pending.pop(0))
