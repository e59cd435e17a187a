"""ctypes binding of ``csrc/libqcur_b200.so`` (the C ABI in include/qcur_b200.h).

This module is the only place Python touches the native library.  Device
memory and streams come from PyTorch (plumbing only): device buffers are
``torch.float64`` CUDA tensors, and every call runs on the caller's current
torch stream.  There is no CPU fallback: without the built library or a CUDA
device, :func:`device` raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import (
    DegenerateDistributionError,
    ParameterError,
    QcurError,
    SamplingError,
    ShapeError,
)

LIB_PATH = Path(__file__).resolve().parent / "csrc" / "libqcur_b200.so"

QCUR_OK = 0
_STATUS_EXC = {
    1: ShapeError,
    2: ParameterError,
    3: DegenerateDistributionError,
    4: SamplingError,
}
STRATEGY_CODES = {"length": 0, "uniform": 1}
CORE_CODES = {"projection": 0, "intersection": 1}
OP_N, OP_H = 0, 1

#: every symbol include/qcur_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "qcur_abi_version", "qcur_create", "qcur_destroy", "qcur_last_error", "qcur_last_info",
    "qcur_set_stream", "qcur_synchronize", "qcur_set_kappa_limit", "qcur_force_robust",
    "qcur_rng_seed", "qcur_rng_advance", "qcur_rng_random",
    "qcur_upload_planar", "qcur_download_planar", "qcur_memcpy",
    "qcur_length_distributions", "qcur_uniform_distributions", "qcur_draw_indices", "qcur_qmcur",
    "qcur_cur_error", "qcur_approx", "qcur_check", "qcur_qgemm", "qcur_pseudoinverse",
    "qcur_frobenius_sq", "qcur_synth_lowrank", "qcur_fp64_peak_tflops", "qcur_int8_peak_tops",
    "qcur_profile", "qcur_profile_read", "qcur_launch_count", "qcur_pairwise_host", "qcur_synth_image",
    "qcur_colsums_seq", "qcur_pairwise_sums", "qcur_vec_div", "qcur_gather_cols", "qcur_gather_rows",
    "qcur_qgemm_ex", "qcur_qgemm_int8", "qcur_qgemm_herm_int8", "qcur_set_gemm_mode", "qcur_qsvd_jacobi", "qcur_qsvd_jacobi_top", "qcur_chol_inv", "qcur_series_l2inv", "qcur_kappa_check", "qcur_factor",
    "qcur_synth_lowrank_rows", "qcur_synth_normals", "qcur_xq", "qcur_complex_adjoint", "qcur_approx_batched", "qcur_colsums_seq_ex", "qcur_series_inv", "qcur_qmcur_ex", "qcur_qmcur_host",
    "qcur_project_observed", "qcur_complete_sweep", "qcur_cur_given", "qcur_qgemv",
    "qcur_upload_length", "qcur_status_async", "qcur_status_map",
    "qcur_graph_begin", "qcur_graph_end", "qcur_graph_launch", "qcur_graph_destroy",
    "qcur_xq_workspace_bytes", "qcur_upload_length_xq", "qcur_qmcur_host_xq",
)

_c_dp = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64p = ctypes.POINTER(ctypes.c_uint64)
_c_dp4 = ctypes.c_void_p * 4
_lib = None
_lib_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    """The sm_100a library or the CUDA device it needs is missing."""


def load_library() -> ctypes.CDLL:
    """Load the in-tree shared library and declare the ABI signatures."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeUnavailable(
                f"{LIB_PATH} is not built; run `python -m paper_2402_19147_b200.build` "
                "(there is no CPU fallback for the QMCUR path)"
            )
        # experiments only: time another build of the library against this one (A/B runs)
        ab = os.environ.get("QCUR_LIB_AB")
        lib = ctypes.CDLL(ab if ab else str(LIB_PATH))
        sig = {
            "qcur_abi_version": (ctypes.c_int, []),
            "qcur_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
            "qcur_destroy": (None, [_c_dp]),
            "qcur_last_error": (ctypes.c_char_p, [_c_dp]),
            "qcur_last_info": (ctypes.c_uint, [_c_dp]),
            "qcur_set_stream": (ctypes.c_int, [_c_dp, _c_dp]),
            "qcur_synchronize": (ctypes.c_int, [_c_dp]),
            "qcur_set_kappa_limit": (ctypes.c_int, [_c_dp, ctypes.c_double]),
            "qcur_force_robust": (ctypes.c_int, [_c_dp, ctypes.c_int]),
            "qcur_rng_seed": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32), ctypes.c_int, _u64p]),
            "qcur_rng_advance": (ctypes.c_int, [_u64p, ctypes.c_uint64]),
            "qcur_rng_random": (ctypes.c_int, [_u64p, _i64, _c_dp]),
            "qcur_upload_planar": (ctypes.c_int, [_c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _i64, _i64, _c_dp]),
            "qcur_download_planar": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _i64, _c_dp, _c_dp, _c_dp, _c_dp]),
            "qcur_memcpy": (ctypes.c_int, [_c_dp, _c_dp, _c_dp, ctypes.c_size_t, ctypes.c_int]),
            "qcur_length_distributions": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp, _c_dp]),
            "qcur_uniform_distributions": (ctypes.c_int, [_c_dp, _i64, _i64, _c_dp, _c_dp]),
            "qcur_draw_indices": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _u64p, _c_dp]),
            "qcur_qmcur": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp, _c_dp, _i64, _i64, _u64p,
                                          _c_dp, _c_dp, _c_dp, _c_dp, _c_dp]),
            "qcur_qmcur_ex": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp, _c_dp, _i64, _i64, _u64p,
                                             ctypes.c_int, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp]),
            "qcur_qmcur_host": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp, _c_dp, _i64, _i64, _u64p,
                                               ctypes.c_int, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp,
                                               _c_dp4, _c_dp4, _c_dp4]),
            "qcur_status_async": (ctypes.c_int, [_c_dp, _c_dp]),
            "qcur_status_map": (ctypes.c_int, [_c_dp, ctypes.c_uint]),
            "qcur_upload_length": (ctypes.c_int, [_c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _i64, _i64, _c_dp, _c_dp, _c_dp]),
            "qcur_xq_workspace_bytes": (ctypes.c_size_t, [_c_dp, _i64, _i64, _i64]),
            "qcur_upload_length_xq": (ctypes.c_int, [_c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _i64, _i64, _i64, _c_dp, _c_dp,
                                                     _c_dp, _c_dp]),
            "qcur_qmcur_host_xq": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp, _c_dp, _i64, _i64, _u64p,
                                                  ctypes.c_int, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp,
                                                  _c_dp4, _c_dp4, _c_dp4, _c_dp]),
            "qcur_qgemv": (ctypes.c_int, [_c_dp, ctypes.c_int, _i64, _i64, _c_dp, _i64, _c_dp, _c_dp]),
            "qcur_cur_given": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp, _i64, _c_dp, _i64, _c_dp, _c_dp, _c_dp]),
            "qcur_project_observed": (ctypes.c_int, [_c_dp, _c_dp, _c_dp, _c_dp, _i64, _i64, _c_dp]),
            "qcur_complete_sweep": (ctypes.c_int, [_c_dp, _c_dp, _c_dp, _c_dp, _i64, _i64, ctypes.c_int, _u64p, _i64,
                                                   _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp]),
            "qcur_cur_error": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp, _i64, _c_dp, _c_dp, _i64, ctypes.c_double,
                                              _c_dp]),
            "qcur_approx": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, ctypes.c_int, _u64p, _i64, _i64,
                                           _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, ctypes.c_double, ctypes.c_int,
                                           _c_dp]),
            "qcur_check": (ctypes.c_int, [_c_dp]),
            "qcur_qgemm": (ctypes.c_int, [_c_dp, ctypes.c_int, ctypes.c_int, _i64, _i64, _i64, ctypes.c_double,
                                          _c_dp, _i64, _c_dp, _i64, ctypes.c_double, _c_dp, _i64]),
            "qcur_pseudoinverse": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, ctypes.c_double, _c_dp]),
            "qcur_frobenius_sq": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, ctypes.POINTER(ctypes.c_double)]),
            "qcur_synth_lowrank": (ctypes.c_int, [_c_dp, _i64, _i64, _i64, ctypes.c_uint64, ctypes.c_double,
                                                  ctypes.c_int, _c_dp]),
            "qcur_fp64_peak_tflops": (ctypes.c_double, [_c_dp]),
            "qcur_int8_peak_tops": (ctypes.c_double, [_c_dp]),
            "qcur_profile": (ctypes.c_int, [_c_dp, ctypes.c_int]),
            "qcur_graph_begin": (ctypes.c_int, [_c_dp]),
            "qcur_graph_end": (ctypes.c_int, [_c_dp, ctypes.POINTER(ctypes.c_void_p)]),
            "qcur_graph_launch": (ctypes.c_int, [_c_dp, _c_dp]),
            "qcur_graph_destroy": (ctypes.c_int, [_c_dp]),
            "qcur_profile_read": (ctypes.c_int, [_c_dp, ctypes.c_char_p, ctypes.c_size_t]),
            "qcur_launch_count": (ctypes.c_ulonglong, []),
            "qcur_pairwise_host": (ctypes.c_int, [_c_dp, _i64, ctypes.POINTER(ctypes.c_double)]),
            "qcur_synth_image": (ctypes.c_int, [_c_dp, _i64, _i64, ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                                                _c_dp]),
            "qcur_colsums_seq": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp, _c_dp, _c_dp]),
            "qcur_pairwise_sums": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _i64, _c_dp]),
            "qcur_vec_div": (ctypes.c_int, [_c_dp, _c_dp, _i64, _c_dp, _c_dp]),
            "qcur_gather_cols": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp, _i64, _c_dp]),
            "qcur_gather_rows": (ctypes.c_int, [_c_dp, _c_dp, _i64, _c_dp, _i64, _c_dp]),
            "qcur_qgemm_ex": (ctypes.c_int, [_c_dp, ctypes.c_int, ctypes.c_int, _i64, _i64, _i64, ctypes.c_double,
                                             _c_dp, _i64, _c_dp, _i64, ctypes.c_double, _c_dp, _i64, ctypes.c_int]),
            "qcur_set_gemm_mode": (ctypes.c_int, [_c_dp, ctypes.c_int]),
            "qcur_qsvd_jacobi": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _i64, _c_dp, _c_dp, _c_dp,
                                                ctypes.POINTER(ctypes.c_int)]),
            "qcur_qsvd_jacobi_top": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _i64, _c_dp, _c_dp, _c_dp, _i64,
                                                    ctypes.POINTER(ctypes.c_int)]),
            "qcur_qgemm_herm_int8": (ctypes.c_int, [_c_dp, _i64, _i64, _i64, _c_dp, _i64, _c_dp, _i64, _c_dp, _i64]),
            "qcur_qgemm_int8": (ctypes.c_int, [_c_dp, _i64, _i64, _i64, _c_dp, _i64, _c_dp, _i64, _c_dp, _i64,
                                                ctypes.c_int]),
            "qcur_chol_inv": (ctypes.c_int, [_c_dp, _c_dp, _i64, _c_dp]),
            "qcur_series_l2inv": (ctypes.c_int, [_c_dp, _c_dp, _i64, _c_dp]),
            "qcur_kappa_check": (ctypes.c_int, [_c_dp, _c_dp, _c_dp, _i64]),
            "qcur_factor": (ctypes.c_int, [_c_dp, _c_dp, ctypes.c_int, _i64, _i64, _c_dp, _c_dp]),
            "qcur_synth_lowrank_rows": (ctypes.c_int, [_c_dp, _i64, _i64, _i64, ctypes.c_uint64, ctypes.c_double,
                                                       _i64, _i64, _c_dp]),
            "qcur_series_inv": (ctypes.c_int, [_c_dp, _c_dp, _i64, _c_dp]),
            "qcur_colsums_seq_ex": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _i64, _c_dp, _c_dp, _c_dp, _i64]),
            "qcur_approx_batched": (ctypes.c_int, [_c_dp, _i64, ctypes.POINTER(ctypes.c_void_p), _i64, _i64,
                                                   ctypes.c_int, _u64p, _i64, _i64, _c_dp, _c_dp, _c_dp, _c_dp,
                                                   _c_dp, ctypes.c_double, ctypes.c_int, _c_dp, ctypes.c_int]),
            "qcur_complex_adjoint": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _c_dp]),
            "qcur_xq": (ctypes.c_int, [_c_dp, _c_dp, _i64, _i64, _i64, _c_dp, _i64, _c_dp]),
            "qcur_synth_normals": (ctypes.c_int, [_c_dp, ctypes.c_uint64, ctypes.c_uint64, _i64, _i64,
                                                  ctypes.c_double, _c_dp]),
        }
        for name, (res, args) in sig.items():
            if ab and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


# ---------------------------------------------------------------------------
# numpy-compatible RNG state (host side of pcg64.h)
# ---------------------------------------------------------------------------
def seed_words(seed: int) -> np.ndarray:
    """Little-endian 32-bit words of a non-negative integer seed, as numpy's
    SeedSequence consumes them (seed 0 -> [0])."""
    seed = int(seed)
    if seed < 0:
        raise ValueError("expected non-negative integer")
    words = []
    while True:
        words.append(seed & 0xFFFFFFFF)
        seed >>= 32
        if seed == 0:
            break
    return np.array(words, dtype=np.uint32)


def state_from_seed(seed: int) -> np.ndarray:
    lib = load_library()
    w = seed_words(seed)
    st = np.zeros(4, dtype=np.uint64)
    rc = lib.qcur_rng_seed(w.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), int(w.size),
                           st.ctypes.data_as(_u64p))
    if rc != QCUR_OK:
        raise ParameterError(f"bad seed {seed!r}")
    return st


def state_from_generator(rng: np.random.Generator) -> np.ndarray:
    bg = rng.bit_generator
    s = bg.state
    if s.get("bit_generator") != "PCG64":
        raise ParameterError(f"only PCG64 generators are supported, got {s.get('bit_generator')}")
    state, inc = int(s["state"]["state"]), int(s["state"]["inc"])
    m64 = (1 << 64) - 1
    return np.array([state >> 64, state & m64, inc >> 64, inc & m64], dtype=np.uint64)


def store_generator_state(rng: np.random.Generator, st: np.ndarray) -> None:
    """Write an advanced PCG64 state back, keeping the generator's uint32 buffer."""
    bg = rng.bit_generator
    s = bg.state
    s["state"]["state"] = (int(st[0]) << 64) | int(st[1])
    bg.state = s


def rng_random(state: np.ndarray, count: int) -> np.ndarray:
    lib = load_library()
    out = np.empty(int(count), dtype=np.float64)
    lib.qcur_rng_random(state.ctypes.data_as(_u64p), int(count), out.ctypes.data)
    return out


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------
class Device:
    """One native context per (process, CUDA device); calls run on torch's current stream."""

    def __init__(self, index: int = 0):
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the QMCUR path runs only on the GPU (no CPU fallback)")
        self.torch = torch
        self.lib = load_library()
        self.index = index
        h = ctypes.c_void_p()
        rc = self.lib.qcur_create(index, ctypes.byref(h))
        if rc != QCUR_OK:
            raise NativeUnavailable(f"qcur_create failed with status {rc}")
        self.handle = h
        self.lock = threading.RLock()

    # -- helpers -----------------------------------------------------------
    def _bind_stream(self):
        s = self.torch.cuda.current_stream(self.index).cuda_stream
        self.lib.qcur_set_stream(self.handle, ctypes.c_void_p(s))

    def check(self, rc: int) -> None:
        if rc == QCUR_OK:
            return
        msg = self.lib.qcur_last_error(self.handle)
        msg = msg.decode() if msg else f"status {rc}"
        raise _STATUS_EXC.get(rc, QcurError)(msg)

    def call(self, name: str, *args):
        with self.lock:
            self._bind_stream()
            rc = getattr(self.lib, name)(self.handle, *args)
        if isinstance(rc, int):
            self.check(rc)
        return rc

    def info(self) -> int:
        return int(self.lib.qcur_last_info(self.handle))

    def profile(self, on) -> None:
        """on: False/0 off, True/1 phase events between direct launches, 2 events captured into a
        CUDA graph (kept across replays: call profile_read after every replay)."""
        self.call("qcur_profile", int(on) if not isinstance(on, bool) else (1 if on else 0))

    def profile_read(self) -> dict[str, tuple[float, int]]:
        """{phase: (total_ms, count)} accumulated since profile(True)."""
        buf = ctypes.create_string_buffer(8192)
        self.call("qcur_profile_read", buf, len(buf))
        out = {}
        for item in buf.value.decode().split(";"):
            if item:
                name, ms, cnt = item.split(":")
                out[name] = (float(ms), int(cnt))
        return out

    def launches(self) -> int:
        return int(self.lib.qcur_launch_count())

    def empty_q(self, m: int, n: int):
        """Uninitialised interleaved quaternion matrix (m, n, 4) float64 on the device."""
        return self.torch.empty((int(m), int(n), 4), dtype=self.torch.float64, device=f"cuda:{self.index}")

    def empty(self, *shape, dtype=None):
        dtype = dtype or self.torch.float64
        return self.torch.empty(shape, dtype=dtype, device=f"cuda:{self.index}")

    def pinned_planes(self, m: int, n: int) -> list:
        """Four (m, n) float64 host planes in one page-locked block (torch's caching
        host allocator, so repeated calls reuse the block).  D2H into pinned memory
        runs at full PCIe rate and never page-faults."""
        block = self.torch.empty((4, int(m), int(n)), dtype=self.torch.float64, pin_memory=True)
        return [block[k].numpy() for k in range(4)]

    def pinned_vec(self, count: int, dtype=None):
        return self.torch.empty(int(count), dtype=dtype or self.torch.int64, pin_memory=True).numpy()

    def upload_planes(self, planes) -> "object":
        a0, a1, a2, a3 = (np.ascontiguousarray(p, dtype=np.float64) for p in planes)
        m, n = a0.shape
        out = self.empty_q(m, n)
        self.call("qcur_upload_planar", a0.ctypes.data, a1.ctypes.data, a2.ctypes.data, a3.ctypes.data,
                  m, n, out.data_ptr())
        return out

    def download_planes(self, x, m: int | None = None, n: int | None = None, pinned_out=None):
        m = int(x.shape[0]) if m is None else m
        n = int(x.shape[1]) if n is None else n
        planes = pinned_out if pinned_out is not None else self.pinned_planes(m, n)
        self.call("qcur_download_planar", x.data_ptr(), m, n, n, *(p.ctypes.data for p in planes))
        return planes

    def synchronize(self) -> None:
        self.torch.cuda.synchronize(self.index)


_devices: dict[int, Device] = {}
_dev_lock = threading.Lock()


def device(index: int | None = None) -> Device:
    """The process-wide native context for a CUDA device (created on first use)."""
    if index is None:
        import torch

        index = torch.cuda.current_device() if torch.cuda.is_available() else 0
    with _dev_lock:
        d = _devices.get(index)
        if d is None:
            d = Device(index)
            _devices[index] = d
        return d
