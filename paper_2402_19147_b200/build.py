"""Build the in-tree sm_100a shared library ``csrc/libqcur_b200.so``.

Plain nvcc (no JIT cache): the built .so lives next to the sources so it
travels with the repo snapshot to the GPU box.  Invoked by
``__graft_entry__.build()`` and ``python -m paper_2402_19147_b200.build``.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = CSRC / "libqcur_b200.so"
STAMP = CSRC / "libqcur_b200.so.sha256"  # hash of the sources + flags the library was built from
SOURCES = ["qcur_abi.cu", "k_norms.cu", "k_draw.cu", "k_layout.cu", "k_qgemm.cu", "k_dense.cu", "k_synth.cu",
           "k_chol_cluster.cu", "k_gemv.cu", "k_ozaki.cu", "k_ozaki_err.cu", "k_qsvd.cu", "k_robust.cu", "k_qgemm_small.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-cudart", "static"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    return "nvcc"


def source_hash() -> str:
    """sha256 over every source, header and the compile flags (not mtimes: a copied tree keeps a
    stale library's mtime newer than its sources, so time stamps cannot prove freshness)."""
    h = hashlib.sha256(" ".join(SOURCES + ARCH + FLAGS).encode())
    deps = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h"))
    deps.append(HERE.parent / "include" / "qcur_b200.h")
    for p in deps:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def build_info() -> dict:
    """Which binary the package loads: its path, the source hash it was built from and
    whether that hash matches the sources in the tree."""
    stamp = STAMP.read_text().strip() if STAMP.exists() else None
    return {"lib": str(LIB), "exists": LIB.exists(), "built_from": stamp, "fresh": stamp == source_hash()}


def build(verbose: bool = False, jobs: int | None = None, force: bool = False) -> Path:
    objdir = CSRC / "build"
    objdir.mkdir(exist_ok=True)
    want = source_hash()
    if not force and LIB.exists() and STAMP.exists() and STAMP.read_text().strip() == want:
        return LIB
    procs = []
    objs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        objs.append(obj)
        cmd = [nvcc(), *ARCH, *FLAGS, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((src, out.decode(errors="replace")))
        elif verbose and out:
            print(out.decode(errors="replace"))
    if failed:
        msg = "\n".join(f"--- {s} ---\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)]
    subprocess.run(cmd, check=True)
    STAMP.write_text(want + "\n")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
