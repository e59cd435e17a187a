"""ORACLE — CPU restatement of the reference QMCUR path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU baseline —
never as part of the product path (paper_2402_19147_b200 never imports it).

It restates, in numpy, the algorithm of the reference package ``qcur``
(pkg/src/qcur/) for the path north_star names:

  length_distributions   cur.py:132-150   (numpy sums: order pinned by numpy_order.c)
  uniform_distributions  cur.py:153-157
  default_sample_counts  cur.py:160-172
  draw_indices           cur.py:202-242   (sequential cumsum + searchsorted 'right')
  plan_indices           cur.py:245-254   (one default_rng stream, columns first)
  pseudoinverse          linalg.py:346-362 (cutoff eps*max(m,n)*sigma_max), computed
                         here as pinv of the complex adjoint chi(A) (linalg.py:151-175):
                         chi is a *-homomorphism, so pinv(chi(A)) = chi(pinv(A)) and
                         chi's singular values are A's, each twice -> same cutoff.
  qmcur                  cur.py:257-269   U = pinv(C) @ X @ pinv(R)
  quaternion matmul      quat.py:274-296  (here via the Cayley-Dickson complex pair)
  relative error         cli.py:173-175 / imaging.py:170-177
  singular values        linalg.py:226-310 (qsvd's sigma: chi's values, one per pair)
  numerical_rank         linalg.py:370-378 (the pinv cutoff)
  spectral_norm          linalg.py:365-367 (chi's largest singular value)
  perturbation_bounds    cur.py:306-388   (every quantity is basis-invariant, so W_k, V_k
                         are represented by chi's top-2k singular subspaces: chi(W_k[I,:])
                         spans the same column space as rows I, m+I of that subspace)

Pinned against the live reference (tests/golden/, made by
tests/golden/make_golden.py from /root/reference in the build container).
Third-party algorithms it relies on: numpy 2.3.5 (pairwise summation,
PCG64 + SeedSequence, cumsum, searchsorted) and LAPACK zgesdd via numpy.
"""
from __future__ import annotations

import math

import numpy as np

EPS = float(np.finfo(np.float64).eps)


class OracleError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind  # "shape" | "parameter" | "degenerate" | "sampling"


# ---------------------------------------------------------------------------
# quaternion matrices as 4 planes  <->  Cayley-Dickson complex pair (a, b): A = a + b j
# ---------------------------------------------------------------------------
def to_cd(planes):
    a0, a1, a2, a3 = planes
    return a0 + 1j * a1, a2 + 1j * a3


def from_cd(a, b):
    return (np.ascontiguousarray(a.real), np.ascontiguousarray(a.imag),
            np.ascontiguousarray(b.real), np.ascontiguousarray(b.imag))


def qmatmul(p, q):
    """Quaternion product P Q of plane tuples: (a + b j)(c + d j) = (ac - b conj(d)) + (ad + b conj(c)) j."""
    a, b = to_cd(p)
    c, d = to_cd(q)
    return from_cd(a @ c - b @ np.conj(d), a @ d + b @ np.conj(c))


def conj_t(p):
    a0, a1, a2, a3 = p
    return (a0.T.copy(), -a1.T, -a2.T, -a3.T)


def adjoint(planes):
    """chi(A) = [[a, b], [-conj(b), conj(a)]] (linalg.py:151-164)."""
    a, b = to_cd(planes)
    return np.block([[a, b], [-np.conj(b), np.conj(a)]])


def frob2(planes) -> float:
    return float(sum(np.sum(p * p) for p in planes))


# ---------------------------------------------------------------------------
# sampling
# ---------------------------------------------------------------------------
def length_distributions(planes):
    """Column / row squared-norm weights in numpy's own summation orders."""
    a0, a1, a2, a3 = planes
    sq = ((a0 * a0 + a1 * a1) + a2 * a2) + a3 * a3
    total = float(sq.sum())
    if total <= 0.0:
        raise OracleError("degenerate", "all sampling weights vanish (zero matrix)")
    col = sq.sum(axis=0) / total
    row = sq.sum(axis=1) / total
    return col / col.sum(), row / row.sum()


def uniform_distributions(m: int, n: int):
    if m < 1 or n < 1:
        raise OracleError("parameter", "dimensions must be positive")
    return np.full(n, 1.0 / n), np.full(m, 1.0 / m)


def default_sample_counts(k: int, m: int, n: int):
    if k < 1 or k > min(m, n):
        raise OracleError("parameter", "bad rank")
    c = min(max(k, math.ceil(k * math.log(max(k, 2)))), min(m, n))
    return c, c


def draw_indices(probs, count: int, rng: np.random.Generator) -> np.ndarray:
    """Iterated weighted draw without replacement; one rng.random() per draw."""
    w = np.array(probs, dtype=np.float64, copy=True)
    if count > int(np.count_nonzero(w > 0)):
        raise OracleError("sampling", "not enough positive weights")
    out = np.empty(count, dtype=np.intp)
    last = w.size - 1
    for t in range(count):
        cum = np.cumsum(w)
        if cum[-1] <= 0.0:
            raise OracleError("sampling", "remaining weights sum to zero")
        target = rng.random() * cum[-1]
        k = min(int(np.searchsorted(cum, target, side="right")), last)
        while w[k] == 0.0:
            k -= 1
        out[t] = k
        w[k] = 0.0
    return out


def plan_indices(col_probs, row_probs, num_cols: int, num_rows: int, seed: int):
    rng = np.random.default_rng(int(seed))
    cols = draw_indices(col_probs, num_cols, rng)
    rows = draw_indices(row_probs, num_rows, rng)
    return rows, cols


# ---------------------------------------------------------------------------
# pseudoinverse and the CUR core
# ---------------------------------------------------------------------------
def pinv(planes, tol: float | None = None):
    m, n = planes[0].shape
    chi = adjoint(planes)
    u, s, vh = np.linalg.svd(chi, full_matrices=False)
    smax = float(s[0]) if s.size else 0.0
    if smax == 0.0:
        return tuple(np.zeros((n, m)) for _ in range(4))
    cutoff = EPS * max(m, n) * smax if tol is None else float(tol)
    keep = s > cutoff
    inv = np.zeros_like(s)
    inv[keep] = 1.0 / s[keep]
    p = (vh.conj().T * inv) @ u.conj().T  # 2n x 2m = chi(pinv(A))
    return from_cd(p[:n, :m], p[:n, m:])


def qmcur(planes, col_probs, row_probs, num_cols: int, num_rows: int, seed: int):
    """(rows I, cols J, C, U, R) exactly as cur.py:257-269 defines them."""
    rows, cols = plan_indices(col_probs, row_probs, num_cols, num_rows, seed)
    c = tuple(np.ascontiguousarray(p[:, cols]) for p in planes)
    r = tuple(np.ascontiguousarray(p[rows, :]) for p in planes)
    u = qmatmul(qmatmul(pinv(c), planes), pinv(r))
    return rows, cols, c, u, r


def cur_error(planes, c, u, r):
    """(||X - C U R||_F^2, ||X||_F^2)."""
    recon = qmatmul(qmatmul(c, u), r)
    diff = tuple(x - y for x, y in zip(planes, recon))
    return frob2(diff), frob2(planes)


def approx(planes, strategy: str, rank: int, seed: int, num_cols: int, num_rows: int):
    """make_plan + qmcur + relative error — one unit of the bench metric."""
    m, n = planes[0].shape
    default_sample_counts(rank, m, n)
    if strategy == "length":
        colp, rowp = length_distributions(planes)
    else:
        colp, rowp = uniform_distributions(m, n)
    rows, cols, c, u, r = qmcur(planes, colp, rowp, num_cols, num_rows, seed)
    e2, x2 = cur_error(planes, c, u, r)
    return dict(rows=rows, cols=cols, c=c, u=u, r=r, col_probs=colp, row_probs=rowp,
                rel_err=math.sqrt(e2) / math.sqrt(x2))


def image_u8(planes, scale: float = 255.0):
    """qmat_to_image(scale * X) (imaging.py:90-100): the three imaginary planes,
    clipped to [0, 255] and rounded half to even."""
    return [np.rint(np.clip(scale * p, 0.0, 255.0)).astype(np.uint8) for p in planes[1:]]


def psnr_u8(ref_planes, test_planes, scale: float = 255.0) -> float:
    """imaging.psnr (imaging.py:111-124) of the two decoded images."""
    total = 0.0
    for a, b in zip(image_u8(ref_planes, scale), image_u8(test_planes, scale)):
        d = a.astype(np.float64) - b.astype(np.float64)
        total += float(np.sum(d * d))
    mse = total / (3 * ref_planes[0].shape[0] * ref_planes[0].shape[1])
    return float("inf") if mse == 0.0 else 10.0 * math.log10(255.0 ** 2 / mse)


def rel_fro(a, b) -> float:
    """||a - b||_F / ||b||_F for plane tuples."""
    return math.sqrt(frob2(tuple(x - y for x, y in zip(a, b)))) / math.sqrt(frob2(b))


# ---------------------------------------------------------------------------
# small deterministic generators (element-wise only: identical on every host)
# ---------------------------------------------------------------------------
def random_planes(rng: np.random.Generator, m: int, n: int, scale: float = 1.0):
    return tuple(scale * rng.standard_normal((m, n)) for _ in range(4))


def lowrank_planes(rng: np.random.Generator, m: int, n: int, k: int):
    """P (m x k) Q (k x n) accumulated rank-1 by rank-1 with element-wise numpy
    ops only, so the bits do not depend on the host's BLAS."""
    p = random_planes(rng, m, k)
    q = random_planes(rng, k, n)
    out = [np.zeros((m, n)) for _ in range(4)]
    for t in range(k):
        a = [x[:, t:t + 1] for x in p]
        b = [x[t:t + 1, :] for x in q]
        prod = (
            a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
            a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
            a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
            a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0],
        )
        for s in range(4):
            out[s] = out[s] + prod[s]
    return tuple(out)


# ---------------------------------------------------------------------------
# low-rank completion, Algorithm 2 (completion.py) — the first "next" row of SURVEY §8(f)
# ---------------------------------------------------------------------------
def derive_seed(seed: int, *parts) -> int:
    """bench.py:72-80."""
    import hashlib

    text = "\x1f".join(str(p) for p in parts)
    digest = hashlib.blake2b(text.encode("utf-8"), digest_size=8).digest()
    return (int(seed) ^ int.from_bytes(digest, "little")) & ((1 << 64) - 1)


def random_mask(m: int, n: int, missing_ratio: float, seed: int) -> np.ndarray:
    """completion.py:82-98 (boolean observed map)."""
    total = m * n
    count = round(missing_ratio * total)
    observed = np.ones(total, dtype=bool)
    if count:
        observed[np.random.default_rng(seed).permutation(total)[:count]] = False
    return observed.reshape(m, n)


def project_observed(x, observed, y):
    """completion.py:101-111."""
    return tuple(np.where(observed, yp, xp) for xp, yp in zip(x, y))


def stabilized_reconstruct(planes, rows, cols):
    """cur.py:277-286: C pinv(C) X pinv(R) R for given index sets."""
    c = tuple(np.ascontiguousarray(p[:, cols]) for p in planes)
    r = tuple(np.ascontiguousarray(p[rows, :]) for p in planes)
    u = qmatmul(qmatmul(pinv(c), planes), pinv(r))
    return qmatmul(qmatmul(c, u), r)


def complete(y, observed, rank: int, strategy: str = "length", max_iters: int = 200, rel_tol: float = 1e-4,
             index_policy: str = "resample_each_iter", seed: int = 0):
    """completion.py:157-246: alternating CUR approximation + observed-entry re-projection.
    Returns (x_star planes, history list, converged)."""
    m, n = y[0].shape
    current = project_observed(tuple(np.zeros((m, n)) for _ in range(4)), observed, y)
    count = min(rank + 5, m, n)

    def dists(planes):
        return length_distributions(planes) if strategy == "length" else uniform_distributions(m, n)

    fixed = None
    if index_policy == "fixed":
        colp, rowp = dists(current)
        fixed = plan_indices(colp, rowp, count, count, derive_seed(seed, "draw"))
    history = []
    converged = False
    for t in range(max_iters):
        if fixed is not None:
            approx_p = stabilized_reconstruct(current, fixed[0], fixed[1])
        else:
            colp, rowp = dists(current)
            rows, cols, c, u, r = qmcur(current, colp, rowp, count, count, derive_seed(seed, "sweep", t))
            approx_p = qmatmul(qmatmul(c, u), r)
        updated = project_observed(approx_p, observed, y)
        step = math.sqrt(frob2(tuple(a - b for a, b in zip(updated, current))))
        scale = math.sqrt(frob2(current))
        if scale > 0.0:
            rel = step / scale
        elif step <= 1e-15:
            rel = 0.0
        else:
            rel = float("inf")
        history.append(float(rel))
        current = updated
        if rel <= rel_tol:
            converged = True
            break
    return current, history, converged


# ---------------------------------------------------------------------------
# QSVD quantities and the perturbation bounds (linalg.py:226-383, cur.py:306-388)
# ---------------------------------------------------------------------------
def singular_values(planes) -> np.ndarray:
    """qsvd(a).sigma: chi's singular values, one per pair, nonincreasing (linalg.py:253-255)."""
    return np.linalg.svd(adjoint(planes), compute_uv=False)[0::2]


def _rank_from_sigma(sigma, shape, tol=None) -> int:
    smax = float(sigma[0]) if sigma.size else 0.0
    if smax == 0.0:
        return 0
    cutoff = EPS * max(shape) * smax if tol is None else float(tol)
    return int(np.sum(sigma > cutoff))


def numerical_rank(planes, tol=None) -> int:
    return _rank_from_sigma(singular_values(planes), planes[0].shape, tol)


def spectral_norm(planes) -> float:
    return float(np.linalg.svd(adjoint(planes), compute_uv=False)[0])


def _pinv_norm(sigma, shape, norm: str) -> float:
    """||pinv(A)|| from A's singular values (pinv's cutoff, linalg.py:352-362)."""
    smax = float(sigma[0]) if sigma.size else 0.0
    if smax == 0.0:
        return 0.0
    kept = sigma[sigma > EPS * max(shape) * smax]
    return float(1.0 / kept[-1]) if norm == "spectral" else float(np.sqrt(np.sum(1.0 / kept ** 2)))


def perturbation_bounds(x, e, rows, cols, k: int, norm: str = "spectral") -> dict:
    """The eight fields of cur.py:289-303 for clean X (rank k), noise E and index sets I, J."""
    m, n = x[0].shape
    rows, cols = np.asarray(rows), np.asarray(cols)
    if numerical_rank(x) != k:
        raise OracleError("parameter", "x does not have numerical rank k")
    nfun = spectral_norm if norm == "spectral" else (lambda p: math.sqrt(frob2(p)))
    u, s, vh = np.linalg.svd(adjoint(x), full_matrices=False)
    u2, v2 = u[:, :2 * k], vh.conj().T[:, :2 * k]
    w_sub = u2[np.concatenate([rows, m + rows]), :]   # column space of chi(W_k[I, :])
    v_sub = v2[np.concatenate([cols, n + cols]), :]
    sw = np.linalg.svd(w_sub, compute_uv=False)[0::2]
    sv = np.linalg.svd(v_sub, compute_uv=False)[0::2]
    if _rank_from_sigma(sw, (rows.size, k)) < k or _rank_from_sigma(sv, (cols.size, k)) < k:
        raise OracleError("sampling", "sampled rows of the singular factors lost rank")
    xt = tuple(a + b for a, b in zip(x, e))
    recon = stabilized_reconstruct(xt, rows, cols)
    lhs = nfun(tuple(a - b for a, b in zip(x, recon)))
    c = tuple(np.ascontiguousarray(p[:, cols]) for p in x)
    r = tuple(np.ascontiguousarray(p[rows, :]) for p in x)
    noise = nfun(e)
    xrp = nfun(qmatmul(x, pinv(r)))
    cx = nfun(qmatmul(pinv(c), x))
    e_rows = tuple(np.ascontiguousarray(p[rows, :]) for p in e)
    e_cols = tuple(np.ascontiguousarray(p[:, cols]) for p in e)
    bound_a = nfun(e_rows) * xrp + nfun(e_cols) * cx + 3.0 * noise
    wp = _pinv_norm(sw, (rows.size, k), norm)
    vp = _pinv_norm(sv, (cols.size, k), norm)
    return dict(lhs=lhs, bound_a=bound_a, bound_b=noise * (wp + vp + 3.0), noise_norm=noise, xrp_norm=xrp,
                cx_norm=cx, wsub_pinv_norm=wp, vsub_pinv_norm=vp)
