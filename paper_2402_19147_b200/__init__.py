"""paper_2402_19147_b200 — B200-native QMCUR (quaternion matrix CUR, arXiv 2402.19147).

Drop-in for the reference package's QMCUR path (``qcur``: make_plan, qmcur,
cur_reconstruct, draw_indices, plan_indices, length/uniform distributions,
pseudoinverse, qmat_matmul, the error classes and the QMatrix/Quaternion
types), plus the first "next" row: the completion solver (``complete``,
Algorithm 2) with GPU-resident sweeps.  All numerics run in hand-written sm_100a CUDA behind the C ABI in
include/qcur_b200.h; there is no CPU fallback.
"""
from .errors import (
    DegenerateDistributionError,
    DegenerateSamplingError,
    FileFormatError,
    ParameterError,
    QcurError,
    SamplingError,
    ShapeError,
)
from .quat import QMatrix, Quaternion, qmat_conj_transpose, qmat_frobenius_norm, qmat_matmul, read_qmat, write_qmat
from .cur import (
    STRATEGIES,
    CURFactors,
    SamplingPlan,
    cur_psnr,
    cur_reconstruct,
    cur_relative_error,
    default_sample_counts,
    draw_indices,
    length_distributions,
    make_plan,
    plan_indices,
    qmcur,
    qmcur_device,
    stabilized_reconstruct,
    uniform_distributions,
    PerturbationBounds,
    perturbation_bounds,
)
from .linalg import QSVDResult, lowrank_truncate, numerical_rank, pseudoinverse, qsvd, save_qsvd, spectral_norm
from .stream import StreamResult, approx_stream
from .completion import (
    INDEX_POLICIES,
    CompletionConfig,
    CompletionResult,
    ObservationMask,
    complete,
    derive_seed,
    project_observed,
    random_mask,
)

__all__ = [
    "QcurError", "ShapeError", "ParameterError", "FileFormatError", "DegenerateDistributionError",
    "SamplingError", "DegenerateSamplingError",
    "QMatrix", "Quaternion", "qmat_matmul", "qmat_conj_transpose", "qmat_frobenius_norm",
    "STRATEGIES", "SamplingPlan", "CURFactors", "length_distributions", "uniform_distributions",
    "default_sample_counts", "make_plan", "draw_indices", "plan_indices", "qmcur", "cur_reconstruct",
    "cur_relative_error", "cur_psnr", "qmcur_device", "pseudoinverse", "stabilized_reconstruct",
    "INDEX_POLICIES", "ObservationMask", "CompletionConfig", "CompletionResult", "random_mask", "project_observed",
    "complete", "derive_seed", "read_qmat", "write_qmat", "spectral_norm",
    "StreamResult", "approx_stream",
    "QSVDResult", "qsvd", "numerical_rank", "lowrank_truncate", "save_qsvd", "PerturbationBounds",
    "perturbation_bounds",
]
__version__ = "0.1.0"
