"""Generate tests/golden/golden.npz from the REFERENCE package (qcur).

Run in the build container only (the reference is not on the GPU box):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
It imports /root/reference/pkg/src read-only, runs the reference's own
make_plan / qmcur / cur_reconstruct / draw_indices / length_distributions /
pseudoinverse on the inputs defined in cases.py, and stores the outputs.
"""
from __future__ import annotations

import hashlib
import os
import sys

sys.dont_write_bytecode = True
os.environ.setdefault("QCUR_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import cases  # noqa: E402
import qcur  # noqa: E402  (the reference)


def planes_hash(planes) -> str:
    h = hashlib.sha256()
    for p in planes:
        h.update(np.ascontiguousarray(p, dtype="<f8").tobytes())
    return h.hexdigest()


def main() -> None:
    out = {}
    for name, case in cases.QMCUR_CASES.items():
        m, n, k, noise, gseed, strategy, pseed, nr, nc = case
        x = qcur.QMatrix(*cases.qmcur_input(case))
        plan = qcur.make_plan(x, strategy, k, pseed, num_rows=nr, num_cols=nc)
        f = qcur.qmcur(x, plan)
        diff = x - qcur.cur_reconstruct(f)
        rel = qcur.qmat_frobenius_norm(diff) / qcur.qmat_frobenius_norm(x)
        out[f"{name}/col_probs"] = plan.col_probs
        out[f"{name}/row_probs"] = plan.row_probs
        out[f"{name}/cols"] = f.col_indices.astype(np.int64)
        out[f"{name}/rows"] = f.row_indices.astype(np.int64)
        out[f"{name}/u"] = f.u.to_array()
        out[f"{name}/rel_err"] = np.array([rel])
        out[f"{name}/c_sha"] = np.array([planes_hash(f.c.planes)])
        out[f"{name}/r_sha"] = np.array([planes_hash(f.r.planes)])
        print(name, "rel_err %.6e" % rel)
    for name, case in cases.DIST_CASES.items():
        col, row = qcur.length_distributions(qcur.QMatrix(*cases.dist_input(case)))
        out[f"{name}/col"] = col
        out[f"{name}/row"] = row
    for name, case in cases.DRAW_CASES.items():
        p, count, seed = cases.draw_input(case)
        out[f"{name}/idx"] = qcur.draw_indices(p, count, seed).astype(np.int64)
    for name, case in cases.PINV_CASES.items():
        out[f"{name}/pinv"] = qcur.pseudoinverse(qcur.QMatrix(*cases.pinv_input(case))).to_array()
    from qcur.bench import derive_seed
    from qcur.completion import CompletionConfig, ObservationMask, complete, random_mask

    for name, case in cases.COMPLETION_CASES.items():
        m, n, k, gseed, ratio, mseed, strategy, policy, seed, iters, tol = case
        truth, observed, y = cases.completion_input(case)
        mask = random_mask(m, n, ratio, mseed)
        assert np.array_equal(mask.observed, observed)
        res = complete(qcur.QMatrix(*y), ObservationMask(observed),
                       CompletionConfig(rank=k, strategy=strategy, max_iters=iters, rel_tol=tol,
                                        index_policy=policy, seed=seed))
        out[f"{name}/mask"] = mask.observed
        out[f"{name}/history"] = np.array(res.rel_change_history)
        out[f"{name}/converged"] = np.array([res.converged])
        out[f"{name}/x_star"] = res.x_star.to_array()
        print(name, res.iterations_run, res.converged, res.rel_change_history[-1])
    from qcur.linalg import spectral_norm as ref_spectral_norm
    from qcur.quat import write_qmat as ref_write_qmat

    for name, case in cases.SPECTRAL_CASES.items():
        out[f"{name}/sigma"] = np.array([ref_spectral_norm(qcur.QMatrix(*cases.spectral_input(case)))])
    from qcur.cur import perturbation_bounds as ref_perturbation_bounds
    from qcur.linalg import numerical_rank as ref_numerical_rank
    from qcur.linalg import qsvd as ref_qsvd

    for name, case in cases.QSVD_CASES.items():
        a = qcur.QMatrix(*cases.qsvd_input(case))
        out[f"{name}/sigma"] = np.asarray(ref_qsvd(a).sigma)
        out[f"{name}/rank"] = np.array([ref_numerical_rank(a)])
    for name, case in cases.PERT_CASES.items():
        x, e, rows, cols = cases.pert_input(case)
        b = ref_perturbation_bounds(qcur.QMatrix(*x), qcur.QMatrix(*e), rows, cols, case[2], norm=case[7])
        out[f"{name}/fields"] = np.array([b.lhs, b.bound_a, b.bound_b, b.noise_norm, b.xrp_norm, b.cx_norm,
                                          b.wsub_pinv_norm, b.vsub_pinv_norm])
        print(name, b)
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "x.qmat")
        ref_write_qmat(qcur.QMatrix(*cases.spectral_input(cases.SPECTRAL_CASES["s_1x5"])), path)
        out["qmat/s_1x5_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    out["derive_seed"] = np.array([derive_seed(s, *parts) for s, parts in cases.DERIVE_SEED_CASES], dtype=np.uint64)
    for s in cases.RNG_SEEDS:
        out[f"rng/{s}"] = np.random.default_rng(s).random(8)
    out["meta/numpy"] = np.array([np.__version__])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
