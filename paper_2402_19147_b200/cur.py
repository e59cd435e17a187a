"""QMCUR — the reference's Algorithm-1 entry points, running on the B200.

Drop-in mirror of ``qcur.cur`` for the hot path (pkg/src/qcur/cur.py:39-274):
same names, signatures, return types, validation and exceptions.  Every
numeric step runs on the GPU through the C ABI (include/qcur_b200.h):

  make_plan            cur.py:175-199  -> qcur_length_distributions (K1, numpy-bit-exact)
  draw_indices         cur.py:202-242  -> qcur_draw_indices          (K2, index-exact)
  plan_indices         cur.py:245-254  -> (same, one PCG64 stream, columns first)
  qmcur                cur.py:257-269  -> qcur_qmcur  (K2+K3 gathers+pinv+U on DMMA)
  cur_reconstruct      cur.py:272-274  -> qcur_qgemm x2
  cur_relative_error   (callers cli.py:173-175, imaging.py:170-177) -> qcur_cur_error,
                       fused ||X - CUR||_F without materialising CUR.

Host code here only validates arguments and moves data.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import (
    DegenerateDistributionError,  # noqa: F401  (re-exported for drop-in imports)
    ParameterError,
    SamplingError,
    ShapeError,
)
from .quat import QMatrix, as_planes, from_device, to_device

__all__ = [
    "STRATEGIES",
    "SamplingPlan",
    "CURFactors",
    "length_distributions",
    "uniform_distributions",
    "default_sample_counts",
    "make_plan",
    "draw_indices",
    "plan_indices",
    "qmcur",
    "cur_reconstruct",
    "cur_relative_error",
    "cur_psnr",
    "qmcur_device",
    "stabilized_reconstruct",
    "PerturbationBounds",
    "perturbation_bounds",
]

STRATEGIES = ("length", "uniform")


def _check_strategy(strategy: str) -> str:
    if strategy not in STRATEGIES:
        raise ParameterError(f"strategy must be one of {STRATEGIES}, got {strategy!r}")
    return strategy


def _validated_probs(p, name: str) -> np.ndarray:
    arr = np.asarray(p, dtype=np.float64)
    if arr.ndim != 1 or arr.size == 0:
        raise ShapeError(f"{name} must be a non-empty 1-D array")
    if np.any(arr < 0) or not np.all(np.isfinite(arr)):
        raise ParameterError(f"{name} must be finite and nonnegative")
    total = arr.sum()
    if abs(total - 1.0) > 1e-12:
        raise ParameterError(f"{name} must sum to 1 (got {total!r})")
    return arr


@dataclass(frozen=True)
class SamplingPlan:
    """Strategy, target rank, sample counts |I| = num_rows, |J| = num_cols, seed
    and the two sampling distributions (cur.py:76-107)."""

    strategy: str
    rank: int
    num_rows: int
    num_cols: int
    seed: int
    row_probs: np.ndarray = field(repr=False)
    col_probs: np.ndarray = field(repr=False)

    def __post_init__(self) -> None:
        _check_strategy(self.strategy)
        if self.rank < 1:
            raise ParameterError(f"rank must be positive, got {self.rank}")
        if self.num_rows < self.rank or self.num_cols < self.rank:
            raise ParameterError(
                f"sample counts ({self.num_rows}, {self.num_cols}) must be >= rank {self.rank}"
            )
        rp = _validated_probs(self.row_probs, "row_probs")
        cp = _validated_probs(self.col_probs, "col_probs")
        if rp is self.row_probs:
            rp = rp.copy()
        if cp is self.col_probs:
            cp = cp.copy()
        rp.setflags(write=False)
        cp.setflags(write=False)
        object.__setattr__(self, "row_probs", rp)
        object.__setattr__(self, "col_probs", cp)
        if self.num_rows > rp.size or self.num_cols > cp.size:
            raise ParameterError("sample counts exceed the available indices")


@dataclass(frozen=True)
class CURFactors:
    """C = X[:, J], R = X[I, :], U = pinv(C) X pinv(R) (cur.py:110-129)."""

    row_indices: np.ndarray
    col_indices: np.ndarray
    c: QMatrix
    u: QMatrix
    r: QMatrix

    def __post_init__(self) -> None:
        for name in ("row_indices", "col_indices"):
            idx = np.array(getattr(self, name), dtype=np.intp)
            idx.setflags(write=False)
            object.__setattr__(self, name, idx)
        if tuple(self.u.shape) != (self.col_indices.size, self.row_indices.size):
            raise ShapeError(
                f"U has shape {tuple(self.u.shape)}, expected "
                f"({self.col_indices.size}, {self.row_indices.size})"
            )


# ---------------------------------------------------------------------------
def _to_dev_vec(dev, arr: np.ndarray):
    return dev.torch.from_numpy(np.array(arr, dtype=np.float64, copy=True)).to(f"cuda:{dev.index}")


def length_distributions(x, _xq_rows: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Squared-norm weights (col_probs, row_probs), bit-identical to the
    reference's numpy evaluation (cur.py:132-150).

    Raises DegenerateDistributionError for the zero matrix.  (_xq_rows: make_plan's row count; when
    the later qmcur takes the INT8 X Q_R, the residues of X are formed while X uploads.)"""
    dev = _native.device()
    m, n = (int(v) for v in x.shape)
    col = dev.empty(n)
    row = dev.empty(m)
    if isinstance(x, QMatrix) and (x._dev is None or x._dev[0] is not dev):
        # first use of a host matrix: upload and column pass pipelined (qcur_upload_length);
        # the device copy stays cached on x for qmcur / the error that follow
        a0, a1, a2, a3 = (np.ascontiguousarray(p, dtype=np.float64) for p in x.planes)
        xd = dev.empty_q(m, n)
        ws = None
        if _xq_rows is not None and 0 < int(_xq_rows) <= m:
            with dev.lock:
                nb = int(dev.lib.qcur_xq_workspace_bytes(dev.handle, m, n, int(_xq_rows)))
            if nb > 0:
                ws = dev.empty(nb, dtype=dev.torch.uint8)
        if ws is not None:
            dev.call("qcur_upload_length_xq", a0.ctypes.data, a1.ctypes.data, a2.ctypes.data, a3.ctypes.data, m, n,
                     int(_xq_rows), xd.data_ptr(), col.data_ptr(), row.data_ptr(), ws.data_ptr())
            x._xq = (dev, int(_xq_rows), ws)
        else:
            dev.call("qcur_upload_length", a0.ctypes.data, a1.ctypes.data, a2.ctypes.data, a3.ctypes.data, m, n,
                     xd.data_ptr(), col.data_ptr(), row.data_ptr())
            x._xq = None
        x._dev = (dev, xd)
    else:
        xd = to_device(x, dev)
        dev.call("qcur_length_distributions", xd.data_ptr(), m, n, col.data_ptr(), row.data_ptr())
    return col.cpu().numpy(), row.cpu().numpy()


def uniform_distributions(m: int, n: int) -> tuple[np.ndarray, np.ndarray]:
    """Flat weights 1/n per column and 1/m per row (cur.py:153-157)."""
    if m < 1 or n < 1:
        raise ParameterError(f"dimensions must be positive, got ({m}, {n})")
    dev = _native.device()
    col = dev.empty(int(n))
    row = dev.empty(int(m))
    dev.call("qcur_uniform_distributions", int(m), int(n), col.data_ptr(), row.data_ptr())
    return col.cpu().numpy(), row.cpu().numpy()


def default_sample_counts(k: int, m: int, n: int) -> tuple[int, int]:
    """|I| = |J| = min(max(k, ceil(k ln k)), min(m, n)) (cur.py:160-172)."""
    if k < 1:
        raise ParameterError(f"k must be positive, got {k}")
    if k > min(m, n):
        raise ParameterError(f"k={k} exceeds min(m, n)={min(m, n)}")
    grown = math.ceil(k * math.log(max(k, 2)))
    count = min(max(k, grown), min(m, n))
    return count, count


def make_plan(x, strategy: str, rank: int, seed: int, num_rows: int | None = None,
              num_cols: int | None = None) -> SamplingPlan:
    """SamplingPlan for x with defaulted sample counts (cur.py:175-199)."""
    _check_strategy(strategy)
    m, n = (int(v) for v in x.shape)
    d_rows, d_cols = default_sample_counts(rank, m, n)
    if strategy == "length":
        col_probs, row_probs = length_distributions(x, _xq_rows=num_rows if num_rows is not None else d_rows)
    else:
        col_probs, row_probs = uniform_distributions(m, n)
    return SamplingPlan(
        strategy=strategy,
        rank=rank,
        num_rows=num_rows if num_rows is not None else d_rows,
        num_cols=num_cols if num_cols is not None else d_cols,
        seed=int(seed),
        row_probs=row_probs,
        col_probs=col_probs,
    )


def draw_indices(probs, count: int, seed) -> np.ndarray:
    """``count`` distinct indices by iterated weighted selection (cur.py:202-242).

    ``seed`` is an int or a numpy ``Generator`` (PCG64); a Generator is
    advanced by exactly ``count`` doubles, as the reference consumes it."""
    p = np.array(probs, dtype=np.float64, copy=True)
    if p.ndim != 1 or p.size == 0:
        raise ShapeError("probs must be a non-empty 1-D array")
    if np.any(p < 0) or not np.all(np.isfinite(p)):
        raise ParameterError("probs must be finite and nonnegative")
    count = int(count)
    if count < 1:
        raise ParameterError(f"count must be positive, got {count}")
    positive = int(np.count_nonzero(p > 0))
    if count > positive:
        raise SamplingError(f"cannot draw {count} distinct indices from {positive} positive weights")
    gen = seed if isinstance(seed, np.random.Generator) else None
    state = _native.state_from_generator(gen) if gen is not None else _native.state_from_seed(int(seed))
    dev = _native.device()
    pd = _to_dev_vec(dev, p)
    out = dev.empty(count, dtype=dev.torch.int64)
    dev.call("qcur_draw_indices", pd.data_ptr(), p.size, count, state.ctypes.data_as(_native._u64p),
             out.data_ptr())
    if gen is not None:
        _native.store_generator_state(gen, state)
    return out.cpu().numpy().astype(np.intp)


def plan_indices(plan: SamplingPlan) -> tuple[np.ndarray, np.ndarray]:
    """(row_indices, col_indices) of a plan: columns first, then rows, from one
    stream seeded by plan.seed (cur.py:245-254)."""
    rng = np.random.default_rng(plan.seed)
    col_indices = draw_indices(plan.col_probs, plan.num_cols, rng)
    row_indices = draw_indices(plan.row_probs, plan.num_rows, rng)
    return row_indices, col_indices


def _check_plan_shape(x, plan: SamplingPlan) -> tuple[int, int]:
    m, n = (int(v) for v in x.shape)
    if plan.col_probs.size != n or plan.row_probs.size != m:
        raise ShapeError(
            f"plan distributions sized ({plan.row_probs.size}, {plan.col_probs.size}) "
            f"do not match matrix shape ({m}, {n})"
        )
    return m, n


def _check_core(core: str) -> int:
    if core not in _native.CORE_CODES:
        raise ParameterError(f"unknown core mode {core!r}; expected one of {sorted(_native.CORE_CODES)}")
    return _native.CORE_CODES[core]


def qmcur(x, plan: SamplingPlan, core: str = "projection") -> CURFactors:
    """Sampled CUR factorization of x under the given plan (cur.py:257-269).

    core="projection" (the reference): U = pinv(C) X pinv(R).
    core="intersection": U = pinv(X[I, J]) (the classical CUR middle factor,
    no pass over X beyond the gathers)."""
    core_code = _check_core(core)
    m, n = _check_plan_shape(x, plan)
    c, r = int(plan.num_cols), int(plan.num_rows)
    for probs, count in ((plan.col_probs, c), (plan.row_probs, r)):
        positive = int(np.count_nonzero(probs > 0))
        if count > positive:
            raise SamplingError(f"cannot draw {count} distinct indices from {positive} positive weights")
    dev = _native.device()
    xd = to_device(x, dev)
    colp = _to_dev_vec(dev, plan.col_probs)
    rowp = _to_dev_vec(dev, plan.row_probs)
    state = _native.state_from_seed(plan.seed)
    J = dev.empty(c, dtype=dev.torch.int64)
    I = dev.empty(r, dtype=dev.torch.int64)
    C = dev.empty_q(m, c)
    U = dev.empty_q(c, r)
    R = dev.empty_q(r, n)
    # host factors land in pinned planes; C, R and the indices download while U is computed
    hj, hi = dev.pinned_vec(c), dev.pinned_vec(r)
    hc, hu, hr = dev.pinned_planes(m, c), dev.pinned_planes(c, r), dev.pinned_planes(r, n)
    ptrs = [_native._c_dp4(*(p.ctypes.data for p in planes)) for planes in (hc, hu, hr)]
    xq = getattr(x, "_xq", None) if isinstance(x, QMatrix) else None
    if xq is not None and xq[0] is dev and xq[1] == r:
        # the residues of X for the INT8 X Q_R were formed while make_plan uploaded X
        dev.call("qcur_qmcur_host_xq", xd.data_ptr(), m, n, colp.data_ptr(), rowp.data_ptr(), c, r,
                 state.ctypes.data_as(_native._u64p), core_code, J.data_ptr(), I.data_ptr(), C.data_ptr(),
                 U.data_ptr(), R.data_ptr(), hj.ctypes.data, hi.ctypes.data, *ptrs, xq[2].data_ptr())
    else:
        dev.call("qcur_qmcur_host", xd.data_ptr(), m, n, colp.data_ptr(), rowp.data_ptr(), c, r,
                 state.ctypes.data_as(_native._u64p), core_code, J.data_ptr(), I.data_ptr(), C.data_ptr(),
                 U.data_ptr(), R.data_ptr(), hj.ctypes.data, hi.ctypes.data, *ptrs)
    return CURFactors(
        row_indices=hi,
        col_indices=hj,
        c=_wrap_resident(hc, C, dev),
        u=_wrap_resident(hu, U, dev),
        r=_wrap_resident(hr, R, dev),
    )


def _wrap_resident(planes, t, dev) -> QMatrix:
    out = QMatrix._wrap(*planes)
    out._dev = (dev, t)
    return out


def cur_reconstruct(factors: CURFactors) -> QMatrix:
    """C U R (cur.py:272-274), two DMMA GEMMs, downloaded to the host."""
    dev = _native.device()
    c, u, r = factors.c, factors.u, factors.r
    dc, du, dr = to_device(c, dev), to_device(u, dev), to_device(r, dev)
    m, kc = (int(v) for v in c.shape)
    kr, n = (int(v) for v in r.shape)
    if tuple(u.shape) != (kc, kr):
        raise ShapeError(f"inner dimensions disagree: {tuple(c.shape)} @ {tuple(u.shape)} @ {tuple(r.shape)}")
    P = dev.empty_q(m, kr)
    dev.call("qcur_qgemm", 0, 0, m, kr, kc, 1.0, dc.data_ptr(), kc, du.data_ptr(), kr, 0.0, P.data_ptr(), kr)
    out = dev.empty_q(m, n)
    dev.call("qcur_qgemm", 0, 0, m, n, kr, 1.0, P.data_ptr(), kr, dr.data_ptr(), n, 0.0, out.data_ptr(), n)
    return from_device(out, dev)


def _fancy_index(indices, size: int, what: str, axis: int) -> np.ndarray:
    """Indices as numpy fancy indexing along an axis of length `size` resolves them."""
    idx = np.asarray(indices, dtype=np.intp)
    if idx.ndim != 1 or idx.size == 0:
        raise ShapeError(f"{what} selection must be a non-empty 1-D index list")
    bad = (idx < -size) | (idx >= size)
    if bad.any():
        raise IndexError(f"index {int(idx[bad][0])} is out of bounds for axis {axis} with size {size}")
    return np.where(idx < 0, idx + size, idx).astype(np.int64)


def stabilized_reconstruct(x, row_indices, col_indices) -> QMatrix:
    """Two-sided projection C pinv(C) X pinv(R) R for given index sets (cur.py:277-286):
    the qmcur core on the device (qcur_cur_given), then C U R."""
    dev = _native.device()
    m, n = (int(v) for v in x.shape)
    # the reference selects through take_cols / take_rows (quat.py:215-225): a 1-D non-empty
    # index list (else ShapeError), numpy fancy indexing (negative indices wrap, out of range
    # raises IndexError); columns are taken first (cur.py:282-283)
    cols = _fancy_index(col_indices, n, "column", 1)
    rows = _fancy_index(row_indices, m, "row", 0)
    c, r = int(cols.size), int(rows.size)
    xd = to_device(x, dev)
    J = dev.torch.from_numpy(cols).to(device=f"cuda:{dev.index}")
    I = dev.torch.from_numpy(rows).to(device=f"cuda:{dev.index}")
    C, U, R = dev.empty_q(m, c), dev.empty_q(c, r), dev.empty_q(r, n)
    dev.call("qcur_cur_given", xd.data_ptr(), m, n, J.data_ptr(), c, I.data_ptr(), r, C.data_ptr(), U.data_ptr(),
             R.data_ptr())
    return cur_reconstruct(CURFactors(row_indices=rows, col_indices=cols, c=from_device(C, dev),
                                      u=from_device(U, dev), r=from_device(R, dev)))


@dataclass(frozen=True)
class PerturbationBounds:
    """Observed projection error and its two computable upper bounds (cur.py:289-303)."""

    lhs: float
    bound_a: float
    bound_b: float
    noise_norm: float
    xrp_norm: float
    cx_norm: float
    wsub_pinv_norm: float
    vsub_pinv_norm: float


def perturbation_bounds(x, e, row_indices, col_indices, k: int, norm: str = "spectral") -> PerturbationBounds:
    """Projection-error bounds for a clean rank-k X, noise E and index sets I, J (cur.py:306-388).

    Every matrix operation runs on the device: the QSVD of X and the numerical ranks (quaternion
    one-sided Jacobi), the stabilized reconstruction of X + E, the pseudoinverses, the products
    and the spectral norms (Lanczos) or Frobenius norms."""
    from .errors import DegenerateSamplingError
    from .linalg import numerical_rank, pseudoinverse, qsvd, spectral_norm
    from .quat import qmat_frobenius_norm

    if norm not in ("spectral", "frobenius"):
        raise ParameterError(f"norm must be 'spectral' or 'frobenius', got {norm!r}")
    if tuple(x.shape) != tuple(e.shape):
        raise ShapeError(f"noise shape {tuple(e.shape)} does not match matrix shape {tuple(x.shape)}")
    rows = np.asarray(row_indices, dtype=np.intp)
    cols = np.asarray(col_indices, dtype=np.intp)
    if rows.size < k or cols.size < k:
        raise ParameterError("index sets must contain at least k entries")
    rank_x = numerical_rank(x)
    if rank_x != k:
        raise ParameterError(f"x has numerical rank {rank_x}, expected exactly {k}")
    nfun = spectral_norm if norm == "spectral" else qmat_frobenius_norm

    res = qsvd(x, k)
    w_sub = res.w.take_rows(rows)
    v_sub = res.v.take_rows(cols)
    if numerical_rank(w_sub) < k or numerical_rank(v_sub) < k:
        raise DegenerateSamplingError("sampled rows of the singular factors lost rank; bounds are void")

    xt = x + e
    lhs = nfun(x - stabilized_reconstruct(xt, rows, cols))
    c = x.take_cols(cols)
    r = x.take_rows(rows)
    noise = nfun(e)
    xrp = nfun(x @ pseudoinverse(r))
    cx = nfun(pseudoinverse(c) @ x)
    bound_a = nfun(e.take_rows(rows)) * xrp + nfun(e.take_cols(cols)) * cx + 3.0 * noise
    wsub_pinv = nfun(pseudoinverse(w_sub))
    vsub_pinv = nfun(pseudoinverse(v_sub))
    bound_b = noise * (wsub_pinv + vsub_pinv + 3.0)
    return PerturbationBounds(lhs=float(lhs), bound_a=float(bound_a), bound_b=float(bound_b),
                              noise_norm=float(noise), xrp_norm=float(xrp), cx_norm=float(cx),
                              wsub_pinv_norm=float(wsub_pinv), vsub_pinv_norm=float(vsub_pinv))


def cur_relative_error(x, factors: CURFactors) -> float:
    """||X - C U R||_F / ||X||_F, fused on the GPU (CUR never materialised).

    Same value as the reference's callers compute (cli.py:173-175,
    imaging.relative_error, imaging.py:170-177)."""
    dev = _native.device()
    m, n = (int(v) for v in x.shape)
    c, u, r = factors.c, factors.u, factors.r
    kc, kr = int(u.shape[0]), int(u.shape[1])
    if tuple(c.shape) != (m, kc) or tuple(r.shape) != (kr, n):
        raise ShapeError("factors do not match the matrix shape")
    e2, x2, _, _ = _error_stats(x, factors, 0.0)
    if x2 == 0.0:
        raise ParameterError("reference matrix is zero; relative error undefined")
    return math.sqrt(e2) / math.sqrt(x2)


def _error_stats(x, factors: CURFactors, psnr_scale: float) -> tuple[float, float, float, float]:
    dev = _native.device()
    m, n = (int(v) for v in x.shape)
    c, u, r = factors.c, factors.u, factors.r
    kc, kr = int(u.shape[0]), int(u.shape[1])
    if tuple(c.shape) != (m, kc) or tuple(r.shape) != (kr, n):
        raise ShapeError("factors do not match the matrix shape")
    xd, dc, du, dr = to_device(x, dev), to_device(c, dev), to_device(u, dev), to_device(r, dev)
    out4 = dev.empty(4)
    dev.call("qcur_cur_error", xd.data_ptr(), m, n, dc.data_ptr(), kc, du.data_ptr(), dr.data_ptr(), kr,
             float(psnr_scale), out4.data_ptr())
    return tuple(float(v) for v in out4.cpu().numpy())


def psnr_from_stats(u8_sq: float, imag_sq: float, m: int, n: int) -> tuple[float, float]:
    """(u8 PSNR, float PSNR with peak 1) from the fused statistics.

    u8: imaging.psnr (imaging.py:111-124) of qmat_to_image(s X) vs
    qmat_to_image(s CUR): MSE pooled over the 3 channels, peak 255, +inf when
    identical.  float: the same over the imaginary planes without quantisation."""
    denom = 3.0 * m * n
    mse = u8_sq / denom
    p8 = float("inf") if mse == 0.0 else 10.0 * math.log10(255.0 ** 2 / mse)
    msef = imag_sq / denom
    pf = float("inf") if msef == 0.0 else 10.0 * math.log10(1.0 / msef)
    return p8, pf


def cur_psnr(x, factors: CURFactors, scale: float = 255.0) -> tuple[float, float]:
    """PSNR of the CUR reconstruction of an image-like pure quaternion matrix,
    fused on the GPU: (psnr(qmat_to_image(scale X), qmat_to_image(scale CUR)),
    float PSNR at peak 1).  Mirrors imaging.psnr / qmat_to_image
    (imaging.py:90-124) without materialising CUR or the images."""
    _, _, imag_sq, u8_sq = _error_stats(x, factors, scale)
    m, n = (int(v) for v in x.shape)
    return psnr_from_stats(u8_sq, imag_sq, m, n)


# ---------------------------------------------------------------------------
# device-resident fast entry (bench `value`): no host round trip, no sync
# ---------------------------------------------------------------------------
class DeviceApprox:
    """Preallocated outputs for repeated device-resident approximations."""

    def __init__(self, m: int, n: int, c: int, r: int, dev=None):
        self.dev = dev or _native.device()
        d = self.dev
        self.m, self.n, self.c, self.r = m, n, c, r
        self.J = d.empty(c, dtype=d.torch.int64)
        self.I = d.empty(r, dtype=d.torch.int64)
        self.C = d.empty_q(m, c)
        self.U = d.empty_q(c, r)
        self.R = d.empty_q(r, n)
        self.err4 = d.empty(4)

    def run(self, xd, strategy: str, seed: int, psnr_scale: float = 0.0, core: str = "projection",
            graph: bool = False) -> None:
        """One approximation (qcur_approx).  graph=True replays the whole approximation as
        one CUDA graph (captured on the first call with these arguments after a normal run
        of the same shape): the ~45 launches go out as a single submission."""
        if graph:
            key = (xd.data_ptr(), strategy, int(seed), float(psnr_scale), core)
            if getattr(self, "_gkey", None) != key:
                self.run(xd, strategy, seed, psnr_scale, core)  # sizes the workspace (no allocation inside)
                self.capture(xd, strategy, seed, psnr_scale, core)
            if getattr(self, "_gexec", None) is not None:
                self.dev.call("qcur_graph_launch", self._gexec)
            else:
                self._graph.replay()
            self.graph_replays = getattr(self, "graph_replays", 0) + 1
            return
        core_code = _check_core(core)
        state = _native.state_from_seed(seed)
        self.dev.call("qcur_approx", xd.data_ptr(), self.m, self.n, _native.STRATEGY_CODES[_check_strategy(strategy)],
                      state.ctypes.data_as(_native._u64p), self.c, self.r, self.J.data_ptr(), self.I.data_ptr(),
                      self.C.data_ptr(), self.U.data_ptr(), self.R.data_ptr(), float(psnr_scale),
                      core_code, self.err4.data_ptr())

    def capture(self, xd, strategy: str, seed: int, psnr_scale: float = 0.0, core: str = "projection") -> None:
        """Capture one approximation into the graph that run(graph=True) replays (the workspace must
        already be sized by a normal run with these arguments)."""
        torch = self.dev.torch
        key = (xd.data_ptr(), strategy, int(seed), float(psnr_scale), core)
        self.dev.synchronize()
        self._drop_graph()
        before = self.dev.launches()
        if _native_graphs():
            # native capture (qcur_graph_*): node priorities kept in the replays
            if getattr(self, "_cap_stream", None) is None:
                self._cap_stream = torch.cuda.Stream(self.dev.index)
            ex = ctypes.c_void_p()
            with torch.cuda.stream(self._cap_stream):
                self.dev.call("qcur_graph_begin")
                try:
                    self.run(xd, strategy, seed, psnr_scale, core)
                finally:
                    self.dev.call("qcur_graph_end", ctypes.byref(ex))
            self._gexec = ex
        else:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.run(xd, strategy, seed, psnr_scale, core)
            self._graph = g
        self._gkey = key
        self.graph_kernels = self.dev.launches() - before

    def _drop_graph(self) -> None:
        ex = getattr(self, "_gexec", None)
        if ex is not None:
            self.dev.synchronize()
            self.dev.lib.qcur_graph_destroy(ex)
        self._gexec, self._graph = None, None

    def __del__(self):
        try:
            self._drop_graph()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    def check(self) -> None:
        self.dev.call("qcur_check")

    def stats(self) -> tuple[float, float, float, float]:
        return tuple(float(v) for v in self.err4.cpu().numpy())

    def rel_error(self) -> float:
        e2, x2, _, _ = self.stats()
        return math.sqrt(e2) / math.sqrt(x2)

    def psnr(self) -> tuple[float, float]:
        _, _, imag_sq, u8_sq = self.stats()
        return psnr_from_stats(u8_sq, imag_sq, self.m, self.n)


def _native_graphs() -> bool:
    """QCUR_NATIVE_GRAPH=1: DeviceApprox graph replays through the library's own capture (qcur_graph_*:
    kernel nodes carry the main chain's high / the residues' low priority).  Measured the same as
    torch.cuda.CUDAGraph (cfg2 in flight 326.7 vs 325.2, one at a time 292.7 vs 294.6), so off."""
    import os

    return os.environ.get("QCUR_NATIVE_GRAPH", "0") == "1"


class DeviceBatch:
    """Preallocated outputs for repeated batched approximations of same-shape device matrices
    (qcur_approx_batched): the per-matrix make_plan + qmcur loop of the reference's scaling
    experiment (pkg/src/qcur/bench.py:346-351) as one ABI call whose matrices overlap on
    internal lanes; graph=True replays the whole batch as one CUDA graph."""

    def __init__(self, batch: int, m: int, n: int, c: int, r: int, dev=None, lanes: int = 8):
        self.dev = dev or _native.device()
        d = self.dev
        self.batch, self.m, self.n, self.c, self.r, self.lanes = batch, m, n, c, r, lanes
        self.J = d.empty(batch, c, dtype=d.torch.int64)
        self.I = d.empty(batch, r, dtype=d.torch.int64)
        self.C = d.empty(batch, m, c, 4)
        self.U = d.empty(batch, c, r, 4)
        self.R = d.empty(batch, r, n, 4)
        self.err4 = d.empty(batch, 4)

    def run(self, xds, strategy: str, seeds, psnr_scale: float = 0.0, core: str = "projection",
            graph: bool = False) -> None:
        if len(xds) != self.batch or len(seeds) != self.batch:
            raise ShapeError(f"batch of {self.batch} matrices expected, got {len(xds)} / {len(seeds)} seeds")
        if graph:
            key = (tuple(x.data_ptr() for x in xds), strategy, tuple(int(s) for s in seeds), float(psnr_scale), core)
            if getattr(self, "_gkey", None) != key:
                torch = self.dev.torch
                self.run(xds, strategy, seeds, psnr_scale, core)  # sizes every lane's workspace first
                self.dev.synchronize()
                g = torch.cuda.CUDAGraph()
                before = self.dev.launches()
                with torch.cuda.graph(g):
                    self.run(xds, strategy, seeds, psnr_scale, core)
                self._graph, self._gkey = g, key
                self.graph_kernels = self.dev.launches() - before
            self._graph.replay()
            self.graph_replays = getattr(self, "graph_replays", 0) + 1
            return
        core_code = _check_core(core)
        states = np.concatenate([_native.state_from_seed(int(sd)) for sd in seeds]).astype(np.uint64)
        ptrs = (ctypes.c_void_p * self.batch)(*[x.data_ptr() for x in xds])
        self._keep = (states, ptrs)
        self.dev.call("qcur_approx_batched", self.batch, ptrs, self.m, self.n,
                      _native.STRATEGY_CODES[_check_strategy(strategy)], states.ctypes.data_as(_native._u64p),
                      self.c, self.r, self.J.data_ptr(), self.I.data_ptr(), self.C.data_ptr(), self.U.data_ptr(),
                      self.R.data_ptr(), float(psnr_scale), core_code, self.err4.data_ptr(), int(self.lanes))

    def check(self) -> None:
        self.dev.call("qcur_check")

    def rel_errors(self) -> np.ndarray:
        e = self.err4.cpu().numpy()
        return np.sqrt(e[:, 0]) / np.sqrt(e[:, 1])


def qmcur_device(xd, strategy: str, rank: int, seed: int, num_rows: int, num_cols: int) -> DeviceApprox:
    """One whole approximation on a device-resident interleaved X (m, n, 4)."""
    m, n = int(xd.shape[0]), int(xd.shape[1])
    default_sample_counts(rank, m, n)
    out = DeviceApprox(m, n, int(num_cols), int(num_rows))
    out.run(xd, strategy, seed)
    out.check()
    return out
