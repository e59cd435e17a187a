#!/usr/bin/env python
"""QMCUR benchmark (BASELINE.json metric: QMCUR approx/sec at m=n=4000).

One *step* = one complete approximation of the BASELINE cfg2 workload on a
device-resident matrix: length-squared distributions (numpy-bit-exact), the
index draw, C/R gathers, pinv(C), pinv(R), U = pinv(C) X pinv(R) and the fused
relative error ||X - CUR||_F / ||X||_F.  The input (512 MB) is larger than L2,
so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

N > 1 is launched by torchrun, one rank per GPU: cfg1-cfg3 do not shard one
matrix profitably, so ranks run independent replicas (weak
scaling, no data-path collective); timing is the max over ranks.

Rank 0 prints ONE JSON line.  Extra keys: roofline (dominant kernel, live CUDA
events), phases (per-phase ms), step_roofline, cpu_baseline (the oracle port
timed on this host), e2e (public API with pinned host buffers, H2D/D2H inside
the timed region), clocks (NVML sampled during the timed region).
"""
from __future__ import annotations

import argparse
import json
from pathlib import Path
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QMCUR approx/sec at m=n=4000; achieved HBM GB/s and FP64 TFLOP/s vs B200 peak"

CONFIGS = {
    # BASELINE.json configs[0]: 1000x1000, rank 10, N(0, 1e-6) noise (std 1e-3), uniform, c=r=40, seed 0
    "cfg1": dict(m=1000, n=1000, rank=10, noise=1e-3, relative=False, strategy="uniform", c=40, r=40,
                 plan_seed=0, gen_seed=20240229, batch=1),
    # configs[1]: 4000x4000, rank 50, noise 1e-3 relative to ||S||_F, length, c=r=200, seed 1  (the headline)
    "cfg2": dict(m=4000, n=4000, rank=50, noise=1e-3, relative=True, strategy="length", c=200, r=200,
                 plan_seed=1, gen_seed=20240229, batch=1),
    # configs[2]: 2048x2048 image-like pure quaternion (30 separable cosine products per colour plane,
    # quantised to 1/255, + N(0, 0.02^2)), length sampling, c=r in {64, 128, 256} (--c), PSNR reported
    "cfg3": dict(m=2048, n=2048, rank=64, noise=0.02, relative=False, strategy="length", c=128, r=128,
                 plan_seed=3, gen_seed=20240303, batch=1, image=True),
    # configs[4]: 32768x32768 (34.4 GB, generated on device), rank 200, 1e-3 relative noise, length,
    # c=r=1000; the CPU oracle is not run (host RAM / hours)
    "cfg5": dict(m=32768, n=32768, rank=200, noise=1e-3, relative=True, strategy="length", c=1000, r=1000,
                 plan_seed=5, gen_seed=20240305, batch=1, no_cpu=True),
    # configs[3]: batch of 64 1024x1024, rank 20, 1e-4 relative noise, uniform, c=r=80, per-matrix seed b
    "cfg4": dict(m=1024, n=1024, rank=20, noise=1e-4, relative=True, strategy="uniform", c=80, r=80,
                 plan_seed=0, gen_seed=20240301, batch=64),
}


def workload_name(cfg_name: str, cfg: dict) -> str:
    b = f"{cfg['batch']} x " if cfg["batch"] > 1 else ""
    if cfg.get("image"):
        return (f"{cfg_name}: {cfg['m']}x{cfg['n']} image-like pure quaternion (30 separable cosine products per "
                f"plane, quantised 1/255, + N(0, {cfg['noise']:g}^2)), {cfg['strategy']} sampling, c=r={cfg['c']}, "
                f"plan seed {cfg['plan_seed']}")
    return (f"{cfg_name}: {b}{cfg['m']}x{cfg['n']} fp64 quaternion, rank {cfg['rank']} Gaussian factors + "
            f"{'relative ' if cfg['relative'] else ''}noise {cfg['noise']:g}, {cfg['strategy']} sampling, "
            f"c=r={cfg['c']}, plan seed {cfg['plan_seed']}")


def alg_counts(cfg: dict) -> dict:
    """Algorithmic work per approximation."""
    m, n, c, r = cfg["m"], cfg["n"], cfg["c"], cfg["r"]
    length = 1 if cfg["strategy"] == "length" else 0
    return dict(
        flop=32.0 * (c * m * n + c * n * r + m * c * r + m * r * n),
        bytes=32.0 * m * n * (2 + length) + 64.0 * (m * c + r * n),
        gemm_xq_flop=32.0 * m * n * r,
        error_flop=32.0 * m * r * n,
        length_bytes=32.0 * m * n,
        gather_bytes=64.0 * (m * c + r * n),
    )


def ncu_traffic(cfg_name: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    committed `ncu --set full` capture summary (profiles/*_ncu_traffic_<cfg>.json, written by
    tools/ncu_traffic.py); (None, None) when no capture of this config exists."""
    files = sorted(Path(__file__).resolve().parent.glob(f"profiles/*_ncu_traffic_{cfg_name}.json"))
    if not files:
        return None, None
    try:
        d = json.loads(files[-1].read_text())
        return float(d[kernel]["traffic_bytes"]), f"{files[-1].name}: {d[kernel]['kernel']}"
    except (KeyError, TypeError, ValueError):
        return None, None


def committed_dmma_peak():
    """Sustained DMMA peak of this pool's B200 from the committed microbenchmark
    (tools/fp64_peak.cu -> profiles/*fp64_peak_sustained.jsonl); the roofline uses the
    larger of it and the live probe, so a slow live probe cannot inflate `frac`."""
    best = None
    for f in sorted(Path(__file__).resolve().parent.glob("profiles/*fp64_peak_sustained.jsonl")):
        for line in f.read_text().splitlines():
            try:
                d = json.loads(line)
            except ValueError:
                continue
            if str(d.get("test", "")).startswith("dmma"):
                best = max(best or 0.0, float(d["tflops"]))
    return best


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return json.load(fh)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# clocks (NVML) sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x4: "sw_power_cap",
        0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        self.ok = False
        self.samples = []
        self.reasons = set()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("internal_api") in ("openblas", "mkl")]
        if n:
            return int(max(n))
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def host_lowrank(cfg: dict, seed: int):
    """Same shapes / distributions as the device generator, numpy on the host
    (reference arm: no code of ours on its path)."""
    if os.path.join(ROOT, "oracle") not in sys.path:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    m, n, k = cfg["m"], cfg["n"], cfg["rank"]
    g = np.random.default_rng(seed)
    if cfg.get("image"):  # same recipe as qcur_synth_image (numpy RNG instead of Philox)
        y, x = np.arange(m)[:, None] / m, np.arange(n)[None, :] / n
        planes = [np.zeros((m, n))]
        for _ in range(3):
            v = np.zeros((m, n))
            for _ in range(30):
                f = sum(g.standard_normal() / (t + 1) * np.cos(2 * np.pi * (8 * g.random() * y) + 2 * np.pi * g.random())
                        for t in range(3))
                h = sum(g.standard_normal() / (t + 1) * np.cos(2 * np.pi * (8 * g.random() * x) + 2 * np.pi * g.random())
                        for t in range(3))
                v += f * h
            v = (v - v.min()) / (v.max() - v.min())
            planes.append(np.rint(255 * v) / 255 + cfg["noise"] * g.standard_normal((m, n)))
        return tuple(planes)
    p = O.random_planes(g, m, k)
    q = O.random_planes(g, n, k)
    s = O.qmatmul(p, O.conj_t(q))
    if cfg["relative"]:
        sigma = cfg["noise"] * math.sqrt(O.frob2(s) / (4.0 * m * n))
    else:
        sigma = cfg["noise"]
    return tuple(x + sigma * g.standard_normal(x.shape) for x in s)


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def ref_worker(args, cfg_name: str, cfg: dict) -> None:
    """--ref-worker: time the UNMODIFIED reference package (baseline/_ref, installed from
    /root/reference/pkg) through its own public API, in a process whose BLAS thread caps were
    set in the environment before Python started (the reference's _threads.py:4-7 contract).
    One step = make_plan + qmcur (cur.py:175-199, 257-269) + the relative error as its CLI
    computes it (cur_reconstruct, x - recon, qmat_frobenius_norm ratio; cli.py:171-175), for
    every matrix of the config.  Prints one JSON dict for the parent."""
    sys.path.insert(0, REF_DIR)
    import qcur  # noqa: E402  (the reference; nothing of this repository on its path)

    planes = host_lowrank(cfg, cfg["gen_seed"])
    x = qcur.QMatrix(*planes)
    budget_s = float(os.environ.get("QCUR_REF_BUDGET_S", "120"))

    def step(b: int):
        plan = qcur.make_plan(x, cfg["strategy"], cfg["rank"], cfg["plan_seed"] + b, num_rows=cfg["r"],
                              num_cols=cfg["c"])
        f = qcur.qmcur(x, plan)
        recon = qcur.cur_reconstruct(f)
        return float(qcur.qmat_frobenius_norm(x - recon) / qcur.qmat_frobenius_norm(x))

    for _ in range(min(args.warmup, 1)):
        step(0)
    times, err = [], None
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for b in range(cfg["batch"]):
            err = step(b)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget_s:
            break
    print(json.dumps({"times": times, "rel_err": err, "warmup": min(args.warmup, 1),
                      "qcur_file": qcur.__file__, "threads_env": os.environ.get("OPENBLAS_NUM_THREADS")}),
          flush=True)


def reference_subprocess(cfg_name: str, cfg: dict, steps: int, warmup: int, budget_s: float):
    """Run ref_worker in a fresh interpreter with every BLAS thread cap set to the host's cores;
    None when baseline/_ref is not installed."""
    import subprocess

    if not os.path.isdir(os.path.join(REF_DIR, "qcur")):
        return None
    cores = len(os.sched_getaffinity(0))
    env = dict(os.environ)
    for var in ("QCUR_THREADS", "OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        env[var] = str(cores)
    env["QCUR_REF_BUDGET_S"] = str(budget_s)
    cmd = [sys.executable, os.path.abspath(__file__), "--ref-worker", "--config", cfg_name, "--steps", str(steps),
           "--warmup", str(warmup)]
    if cfg_name == "cfg3":
        cmd += ["--c", str(cfg["c"])]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=budget_s * 4 + 600)
    if out.returncode != 0:
        raise RuntimeError(f"reference worker failed: {out.stderr[-2000:]}")
    d = json.loads(out.stdout.strip().splitlines()[-1])
    d["cores"] = cores
    return d


def run_reference(args, cfg_name: str, cfg: dict) -> None:
    """--impl reference: the reference's own CPU implementation of the path on this host.

    The unmodified reference package (baseline/_ref) through its public API, BLAS threads
    capped at the host's cores before its interpreter starts.  The oracle port (oracle/oracle.py,
    the numpy restatement the parity tests use) is timed beside it as a second number; when
    baseline/_ref is absent the port is the arm (kind "port")."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    budget_s = float(os.environ.get("QCUR_REF_BUDGET_S", "120"))
    ref = reference_subprocess(cfg_name, cfg, args.steps, args.warmup, budget_s)

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    planes = host_lowrank(cfg, cfg["gen_seed"])
    cores = cpu_threads()
    port_steps = 2 if ref is not None else args.steps

    def step(b: int):
        return O.approx(planes, cfg["strategy"], cfg["rank"], cfg["plan_seed"] + b, cfg["c"], cfg["r"])["rel_err"]

    for _ in range(min(args.warmup, 1)):
        step(0)
    ptimes = []
    perr = None
    t_all = time.perf_counter()
    for _ in range(port_steps):
        t0 = time.perf_counter()
        for b in range(cfg["batch"]):
            perr = step(b)
        ptimes.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget_s:
            break
    port = {"value": len(ptimes) * cfg["batch"] / sum(ptimes), "unit": "approx/s", "cores": cores, "kind": "port",
            "steps": len(ptimes), "rel_err": perr,
            "sample": "oracle/oracle.py (numpy restatement of the reference path) on the same host input"}
    if ref is not None:
        times = ref["times"]
        kind, cores_used, warm = "reference", ref["cores"], ref["warmup"]
        rel_err = ref["rel_err"]
        sample = (f"{len(times)} of {args.steps} requested steps timed (budget {budget_s:.0f}s), each step = "
                  f"{cfg['batch']} full approximation(s) of {cfg_name} by the unmodified reference package "
                  f"(baseline/_ref: make_plan + qmcur + cur_reconstruct + relative error, cli.py:171-175), "
                  f"BLAS threads = {cores_used}")
    else:
        times, kind, cores_used, warm, rel_err = ptimes, "port", cores, min(args.warmup, 1), perr
        sample = (f"{len(times)} steps of the oracle port (baseline/_ref not installed), each step = "
                  f"{cfg['batch']} full approximation(s) of {cfg_name}")
    elapsed = sum(times)
    value = len(times) * cfg["batch"] / elapsed
    ms = 1e3 * elapsed / len(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "approx/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (numpy host generator)",
        "config": {"workload": workload_name(cfg_name, cfg)}, "rel_err": rel_err,
        "world_size": int(os.environ.get("WORLD_SIZE", "1")),
        "cpu_baseline": {"value": value, "unit": "approx/s", "cores": cores_used, "kind": kind, "sample": sample},
        "port": port,
        "e2e": {"value": value, "unit": "approx/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_rowshard(args, cfg_name: str, cfg: dict, world: int, rank: int, local: int) -> None:
    """One matrix sharded by row blocks across the ranks (cfg5 design):
    each rank generates and keeps its own rows; NCCL collectives carry the
    column-norm chain, subtree totals, R rows, Gram / M all-reduces and error
    partials (paper_2402_19147_b200/rowshard.py).  Strong scaling: one whole
    approximation per step, whatever the number of GPUs."""
    import torch

    from paper_2402_19147_b200 import _native
    from paper_2402_19147_b200.rowshard import Comm, GpuOps, SingleComm, approx_rowsharded
    from paper_2402_19147_b200.sharding import max_over_ranks

    dev = _native.device(local)
    m, n, c, r = cfg["m"], cfg["n"], cfg["c"], cfg["r"]
    rows_b = m // world
    xb = dev.empty_q(rows_b, n)
    dev.call("qcur_synth_lowrank_rows", m, n, cfg["rank"], cfg["gen_seed"], cfg["noise"], rank * rows_b, rows_b,
             xb.data_ptr())
    comm = Comm() if world > 1 else SingleComm()
    ops = GpuOps(dev)
    res = None
    for _ in range(max(args.warmup, 3)):
        res = approx_rowsharded(ops, comm, xb, m, cfg["strategy"], cfg["plan_seed"], c, r)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = dev.launches()
    with sampler:
        e0.record(stream)
        for _ in range(args.steps):
            res = approx_rowsharded(ops, comm, xb, m, cfg["strategy"], cfg["plan_seed"], c, r)
        e1.record(stream)
        torch.cuda.synchronize()
    ms_total = max_over_ranks(e0.elapsed_time(e1), device=f"cuda:{local}")
    # kernels launched in the timed region: direct launches plus the kernels of every graph replay
    launches = dev.launches() - l0  # the sharded step launches directly (no graph replay)
    ms_step = ms_total / args.steps
    counts = alg_counts(cfg)
    peak_live = dev.lib.qcur_fp64_peak_tflops(dev.handle)
    peak_tf = max(peak_live, committed_dmma_peak() or 0.0)
    achieved = counts["flop"] / (ms_step * 1e-3) / 1e12
    if rank == 0:
        line = {
            "metric": METRIC, "value": 1e3 / ms_step, "unit": "approx/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: each rank generates its row block on device (Philox, S = P Q^H on DMMA, noise "
                    "relative to the analytic ||S||_F)",
            "config": {"workload": workload_name(cfg_name, cfg) + " [row-block sharded]", "m": m, "n": n, "c": c,
                       "r": r, "parallelism": f"row blocks of {rows_b} rows x {world} GPUs (NCCL collectives)",
                       "l2": "inputs larger than L2; no flush"},
            "gpu_launches": launches, "rel_err": res["rel_err"],
            "roofline": {"kernel": "whole sharded step (all FP64 GEMMs)", "bound": "tensor",
                         "achieved": achieved / world, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / world / peak_tf, "traffic": None,
                         "peak_source": "FP64 DMMA peak per GPU: max of the live probe and the committed "
                                        "sustained microbenchmark", "peak_live": peak_live},
            "clocks": sampler.summary(),
            "e2e": None, "e2e_note": "row-sharded inputs are generated on device per rank; no host path",
            "cpu_baseline": {"value": None, "unit": "approx/s", "cores": cpu_threads(), "kind": "port",
                             "sample": "not run: the oracle cannot hold a 32768^2 matrix's temporaries"},
        }
        print(json.dumps(line), flush=True)


COMPLETION = dict(m=512, n=768, rank=20, missing=0.5, mask_seed=1, gen_seed=20240229, noise=0.02, sweeps=30,
                  strategy="length", seed=0)


def run_completion(args) -> None:
    """--completion: the first "next" row, Algorithm 2 on a Kodak-sized
    (512 x 768) image-like pure-quaternion matrix with half its entries missing, a fixed number of
    sweeps (rel_tol below reach).  One JSON line, rank 0, 1 GPU."""
    import torch

    from paper_2402_19147_b200 import CompletionConfig, QMatrix, _native, complete, random_mask
    from paper_2402_19147_b200.quat import from_device

    cfgc = dict(COMPLETION)
    m, n = cfgc["m"], cfgc["n"]
    dev = _native.device(0)
    x = dev.empty_q(m, n)
    dev.call("qcur_synth_image", m, n, 30, cfgc["gen_seed"], cfgc["noise"], x.data_ptr())
    truth = from_device(x, dev)
    mask = random_mask(m, n, cfgc["missing"], cfgc["mask_seed"])
    y = QMatrix(*(np.where(mask.observed, p, 0.0) for p in truth.planes))
    cc = CompletionConfig(rank=cfgc["rank"], strategy=cfgc["strategy"], max_iters=cfgc["sweeps"], rel_tol=1e-300,
                          seed=cfgc["seed"])
    res = None
    for _ in range(max(args.warmup, 1)):
        res = complete(y, mask, cc)
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    with sampler:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = complete(y, mask, cc)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
    sweeps_s = args.steps * res.iterations_run / el
    cpu = None
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O

        k = 3
        t0 = time.perf_counter()
        O.complete(tuple(y.planes), mask.observed, cfgc["rank"], cfgc["strategy"], k, 1e-300, "resample_each_iter",
                   cfgc["seed"])
        ct = time.perf_counter() - t0
        cpu = {"value": k / ct, "unit": "sweeps/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"{k} sweeps of the same solve by oracle/oracle.py:complete"}
    err = float(np.sqrt(sum(((a - b) ** 2).sum() for a, b in zip(res.x_star.planes, truth.planes)) /
                        sum((b ** 2).sum() for b in truth.planes)))
    print(json.dumps({
        "metric": "completion sweeps/sec (Algorithm 2, completion.py:157-246)", "value": sweeps_s,
        "unit": "sweeps/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_sweep": 1e3 * el / (args.steps * res.iterations_run), "higher_is_better": True, "dtype": "f64",
        "data": "synthetic image-like pure quaternion (qcur_synth_image), 50% of entries missing (random_mask)",
        "config": {"workload": f"completion {m}x{n}, rank {cfgc['rank']}, {cfgc['strategy']} sampling, "
                               f"{cfgc['sweeps']} sweeps per solve (count = rank + 5 rows / columns)", **cfgc},
        "e2e": {"value": sweeps_s, "unit": "sweeps/s", "api": "complete(y, mask, cfg) on host QMatrix / mask "
                "(upload, all sweeps, x_star download inside the timed region)",
                "h2d_bytes_per_step": 32 * m * n + m * n, "d2h_bytes_per_step": 32 * m * n},
        "rel_err_vs_truth": err, "clocks": sampler.summary(), "cpu_baseline": cpu,
    }))


def run_qsvd(args) -> None:
    """--qsvd: SURVEY 8(f) rank 4, the truncated QSVD comparator (qsvd(x, k), linalg.py:226-310, as the
    reference's scaling experiment races it against QMCUR, bench.py:319-352) on a 1000 x 1000
    rank-10 + noise matrix, k = 10.  CPU baseline: the oracle's complex-adjoint SVD (numpy LAPACK)."""
    import torch

    import paper_2402_19147_b200 as q

    m = n = 1000
    k = 10
    g = np.random.default_rng(20240229)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    # quaternion rank-10 product (on the device GEMM) plus noise
    pf = q.QMatrix(*(g.standard_normal((m, k)) for _ in range(4)))
    qf = q.QMatrix(*(g.standard_normal((k, n)) for _ in range(4)))
    s = pf @ qf
    planes = [a + 1e-3 * g.standard_normal((m, n)) for a in s.planes]
    x = q.QMatrix(*planes)
    res = None
    for _ in range(max(args.warmup, 1)):
        res = q.qsvd(x, k)
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 10))
    sampler = ClockSampler(0)
    with sampler:
        t0 = time.perf_counter()
        for _ in range(steps):
            res = q.qsvd(x, k)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
    recon_err = float((x - res.reconstruct()).frobenius_norm() / x.frobenius_norm())
    cpu = None
    if not args.no_cpu_baseline:
        import oracle as O

        t0 = time.perf_counter()
        _, s_c, _ = np.linalg.svd(O.adjoint(tuple(planes)), full_matrices=False)
        ct = time.perf_counter() - t0
        s_ref = s_c[0::2]
        cpu = {"value": 1.0 / ct, "unit": "qsvd/s", "cores": cpu_threads(), "kind": "port",
               "sample": "the SVD (with vectors) of the 2000 x 2000 complex adjoint, numpy LAPACK zgesdd: the "
                         "dominant step of the reference's qsvd (linalg.py:253), without its Gram-Schmidt pull-back",
               "sigma_rel_diff_top_k": float(np.max(np.abs(s_ref[:k] - res.sigma) / s_ref[0]))}
    print(json.dumps({
        "metric": "truncated QSVD per second (qsvd(x, k), linalg.py:226-310)", "value": steps / el,
        "unit": "qsvd/s", "n_gpus": 1, "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / steps,
        "higher_is_better": True, "dtype": "f64",
        "data": "synthetic host QMatrix: quaternion rank-10 Gaussian product + N(0, 1e-6) noise, seed 20240229",
        "config": {"workload": f"qsvd {m}x{n}, k = {k} (quaternion one-sided Jacobi on the GPU)", "m": m, "n": n,
                   "k": k},
        "e2e": {"value": steps / el, "unit": "qsvd/s", "api": "qsvd(x, k) on a host QMatrix (upload, Jacobi sweeps, "
                "W / sigma / V download inside the timed region)", "h2d_bytes_per_step": 32 * m * n,
                "d2h_bytes_per_step": 32 * (m * n + n * n) + 8 * n},
        "reconstruction_rel_err": recon_err, "jacobi_sweeps": q.linalg._last_sweeps, "clocks": sampler.summary(),
        "cpu_baseline": cpu,
    }))


def spawn_ranks(n: int) -> int:
    """Re-launch this command as n ranks under torch.distributed.run (single node, 127.0.0.1)."""
    import socket
    import subprocess

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c", type=int, default=None, help="override c = r (cfg3: 64, 128 or 256)")
    ap.add_argument("--rowshard", action="store_true",
                    help="shard one matrix by row blocks across the ranks (cfg5 design) instead of replicas")
    ap.add_argument("--qsvd", action="store_true", help="truncated QSVD comparator (SURVEY 8(f) rank 4)")
    ap.add_argument("--ref-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--completion", action="store_true",
                    help="measure the completion solver (Algorithm 2) instead of the QMCUR step")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not args.ref_worker:
        # started as `python bench.py --gpus N`: become N ranks, one per GPU (torchrun on this
        # node, rendezvous on 127.0.0.1); every rank re-enters main() with WORLD_SIZE set
        sys.exit(spawn_ranks(args.gpus))
    if "WORLD_SIZE" in os.environ and not args.ref_worker:
        ws = int(os.environ["WORLD_SIZE"])
        if ws != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch one rank per GPU")
    if args.qsvd:
        run_qsvd(args)
        return
    if args.completion:
        run_completion(args)
        return
    cfg = dict(CONFIGS[args.config])
    if args.c:
        cfg["c"] = cfg["r"] = args.c
    if args.ref_worker:
        ref_worker(args, args.config, cfg)
        return
    if args.impl == "reference":
        run_reference(args, args.config, cfg)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if args.rowshard:
        run_rowshard(args, args.config, cfg, world, rank, local)
        if world > 1:
            dist.destroy_process_group()
        return

    from paper_2402_19147_b200 import _native
    from paper_2402_19147_b200.cur import DeviceApprox, cur_relative_error, make_plan, qmcur
    from paper_2402_19147_b200.quat import QMatrix, drop_device_copy

    dev = _native.device(local)
    m, n, c, r, batch = cfg["m"], cfg["n"], cfg["c"], cfg["r"], cfg["batch"]
    # --- inputs on the device (Philox + DMMA GEMM, deterministic) ---
    # batch configs (cfg4) split the matrices across ranks (no collective, strong
    # scaling); single-matrix configs run one replica per rank (weak scaling)
    from paper_2402_19147_b200.sharding import shard_range

    mine = list(shard_range(batch, world, rank)) if batch > 1 else [0]
    xs = []
    for b in mine:
        x = dev.empty_q(m, n)
        if cfg.get("image"):
            dev.call("qcur_synth_image", m, n, 30, cfg["gen_seed"] + 7919 * rank, cfg["noise"], x.data_ptr())
        else:
            seed_b = cfg["gen_seed"] + 1000 * b + (7919 * rank if batch == 1 else 0)
            dev.call("qcur_synth_lowrank", m, n, cfg["rank"], seed_b, cfg["noise"], 1 if cfg["relative"] else 0,
                     x.data_ptr())
        xs.append(x)
    outs = DeviceApprox(m, n, c, r, dev)
    psnr_scale = 255.0 if cfg.get("image") else 0.0

    use_graph = not os.environ.get("QCUR_NO_GRAPH")
    # Throughput with several independent approximations in flight (single-matrix configs): each
    # lane has its own native context, stream and resident input (a second matrix of the same
    # workload, its own generator seed), so one approximation's latency-bound phases (draws,
    # Cholesky) overlap another's tensor-bound ones.  QCUR_INFLIGHT=1 gives the serial number.
    # in flight: 4 for the small single-matrix configs (cfg1: latency-bound, 2805 -> 4351 approx/s
    # with 4), 2 otherwise (cfg2: 2, 3 and 4 measure the same)
    inflight = int(os.environ.get("QCUR_INFLIGHT", "4" if m * n < 8e6 else "2")) if batch == 1 else 1
    if 32 * m * n > 8e9:  # cfg5: one 34 GB matrix and its workspace fill the GPU; one in flight
        inflight = 1
    lanes = [(dev, outs, xs, torch.cuda.current_stream())]
    for k in range(1, inflight):
        dk = _native.Device(local)
        xk = dk.empty_q(m, n)
        if cfg.get("image"):
            dk.call("qcur_synth_image", m, n, 30, cfg["gen_seed"] + 7919 * rank + 104729 * k, cfg["noise"],
                    xk.data_ptr())
        else:
            dk.call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"] + 7919 * rank + 104729 * k, cfg["noise"],
                    1 if cfg["relative"] else 0, xk.data_ptr())
        lanes.append((dk, DeviceApprox(m, n, c, r, dk), [xk], torch.cuda.Stream(local)))
    lane_pos = [0]

    # batch configs (cfg4): this rank's matrices in one batched ABI call (qcur_approx_batched: the
    # matrices overlap on internal lanes), one CUDA graph replay per step
    bt = None
    if batch > 1:
        from paper_2402_19147_b200.cur import DeviceBatch

        bt = DeviceBatch(len(mine), m, n, c, r, dev, lanes=int(os.environ.get("QCUR_BATCH_LANES", "8")))
        lanes = [(dev, bt, xs, torch.cuda.current_stream())]

    def step(graph=use_graph):
        d_, o_, xs_, st_ = lanes[lane_pos[0] % len(lanes)]
        lane_pos[0] += 1
        with torch.cuda.stream(st_):
            if bt is not None:
                bt.run(xs_, cfg["strategy"], [cfg["plan_seed"] + b for b in mine], psnr_scale, graph=graph)
                return
            for x, b in zip(xs_, mine):
                o_.run(x, cfg["strategy"], cfg["plan_seed"] + b, psnr_scale, graph=graph)

    def replayed():
        return sum(getattr(o_, "graph_replays", 0) * getattr(o_, "graph_kernels", 0) for _, o_, _, _ in lanes)

    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 3) * len(lanes)):
        step()
    for _, o_, _, _ in lanes:
        o_.check()
    torch.cuda.synchronize()

    # --- timed region: device-resident value ---
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = dev.launches() + replayed()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with sampler:
        e0.record(stream)
        for _, _, _, st_ in lanes[1:]:
            st_.wait_event(e0)
        for _ in range(args.steps):
            step()
        for _, _, _, st_ in lanes[1:]:
            stream.wait_stream(st_)
        e1.record(stream)
        torch.cuda.synchronize()
    # kernels launched in the timed region: direct launches plus the kernels of every graph replay
    launches = dev.launches() + replayed() - l0
    if world > 1:
        dist.barrier()
    for _, o_, _, _ in lanes:
        o_.check()
    ms_total = e0.elapsed_time(e1)
    t = torch.tensor([ms_total], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    # units completed by all ranks together / slowest rank's time
    value = (args.steps * batch if batch > 1 else world * args.steps) / (ms_total / 1e3)
    rel_err = float(bt.rel_errors()[-1]) if bt is not None else outs.rel_error()
    # the same loop with one approximation in flight (reported beside the headline)
    serial = None
    if len(lanes) > 1:
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s0.record(stream)
        for _ in range(args.steps):
            outs.run(xs[0], cfg["strategy"], cfg["plan_seed"], psnr_scale, graph=use_graph)
        s1.record(stream)
        torch.cuda.synchronize()
        serial = args.steps / (s0.elapsed_time(s1) / 1e3)

    # --- batch configs: every rank's per-matrix results (error, J, I) assembled on every rank
    # (no collective between approximations, one at the end) ---
    batch_results = None
    if batch > 1:
        from paper_2402_19147_b200.sharding import run_batch_split

        pos = {b: k for k, b in enumerate(mine)}

        def approx_one(b):
            outs.run(xs[pos[b]], cfg["strategy"], cfg["plan_seed"] + b, psnr_scale, graph=False)
            return np.concatenate([[outs.rel_error()], outs.J.cpu().numpy(), outs.I.cpu().numpy()])

        table = run_batch_split(batch, approx_one, 1 + c + r, device=f"cuda:{local}")
        errs = table[:, 0]
        batch_results = {"matrices": int(batch), "rel_err_min": float(errs.min()), "rel_err_max": float(errs.max()),
                         "rel_err_mean": float(errs.mean()),
                         "complete": bool(np.isfinite(table).all()),
                         "gathered_by": "one all-reduce of the (batch, 1 + c + r) table of errors and index sets"}

    # --- phase breakdown (events between phases, same stream), separate pass ---
    dev.profile(True)
    nprof = min(args.steps, 10)
    for _ in range(nprof):
        # one approximation at a time on lane 0 (no other lane in flight), so each phase is timed
        # alone; phase marks are events between direct launches
        with torch.cuda.stream(lanes[0][3]):
            for x, b in zip(xs, mine):
                outs.run(x, cfg["strategy"], cfg["plan_seed"] + b, psnr_scale, graph=False)
        torch.cuda.synchronize()
    phases = dev.profile_read()
    dev.profile(False)
    per_approx = {k: v[0] / max(v[1], 1) for k, v in phases.items()}
    # the same phases as the production path runs them: events captured into the approximation's
    # CUDA graph (external event nodes), harvested after every replay
    graph_phases = None
    if batch == 1:
        try:
            torch.cuda.synchronize()
            gx = xs[0]
            ga = DeviceApprox(m, n, c, r, dev)
            with torch.cuda.stream(lanes[0][3]):
                ga.run(gx, cfg["strategy"], cfg["plan_seed"], psnr_scale)  # sizes the workspace
            torch.cuda.synchronize()
            dev.profile(2)
            with torch.cuda.stream(lanes[0][3]):
                ga.capture(gx, cfg["strategy"], cfg["plan_seed"], psnr_scale)
                for _ in range(nprof):
                    ga.run(gx, cfg["strategy"], cfg["plan_seed"], psnr_scale, graph=True)
                    torch.cuda.synchronize()
                    gph = dev.profile_read()
            dev.profile(False)
            graph_phases = {k: v[0] / max(v[1], 1) for k, v in gph.items()}
            ga._drop_graph()
        except Exception as exc:  # pragma: no cover - measurement extra, never fatal
            dev.profile(False)
            graph_phases = {"unavailable": str(exc)[:200]}
    counts = alg_counts(cfg)
    peak_live = dev.lib.qcur_fp64_peak_tflops(dev.handle)
    peak_tf = max(peak_live, committed_dmma_peak() or 0.0)
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    dom = max(("gemm_xq", "error"), key=lambda k: per_approx.get(k, 0.0))
    # did the dominant product run on the INT8 tensor-core engine? (its extra phase marks say so)
    int8 = ("error_digits" if dom == "error" else "xq_residues") in per_approx
    dom_ms = per_approx.get(dom, float("nan"))
    dom_flop = counts["gemm_xq_flop"] if dom == "gemm_xq" else counts["error_flop"]
    traffic, traffic_src = ncu_traffic(args.config, "gemm_xq" if dom == "gemm_xq" else "error")
    if int8:
        # INT8 kernels: achieved = the tcgen05 kind::i8 multiply-adds the algorithm needs (x2 ops):
        # error = 21 digit products of P (m x 4r) by E(R) (4r x 4n); Y = X Q_R = 15 modular
        # products of X (m x 4n) by E(Q_R) (4n x 4r).  Peak = the live dense kind::i8 probe.
        peak_i8 = dev.lib.qcur_int8_peak_tops(dev.handle)
        i8_ops = 2.0 * (21 if dom == "error" else 15) * m * (4 * r) * (4 * n)
        achieved = i8_ops / (dom_ms * 1e-3) / 1e12
        roofline = {
            "kernel": ("k_oe_err (P R by 21 base-256 digit GEMMs on tcgen05 kind::i8, fused error epilogue)"
                       if dom == "error" else "k_oz_gemm (Y = X Q_R by 15 modular GEMMs on tcgen05 kind::i8)"),
            "bound": "tensor", "achieved": achieved, "peak": peak_i8, "unit": "TOP/s (int8)",
            "frac": achieved / peak_i8 if peak_i8 else None, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": "live dense INT8 probe (qcur_int8_peak_tops: back-to-back tcgen05.mma kind::i8 M128 N256 "
                           "K32, one CTA per SM); MEASURED_PEAKS.json has no INT8 figure",
            "algorithmic_int8_ops_per_launch": i8_ops, "avg_launch_ms": dom_ms,
            "fp64_equivalent_TFps": dom_flop / (dom_ms * 1e-3) / 1e12,
            "fp64_dmma_peak_TFps": peak_tf,
        }
    else:
        achieved = dom_flop / (dom_ms * 1e-3) / 1e12
        roofline = {
            "kernel": "qgemm_kernel<EPI_ERR> (fused C U R + error)" if dom == "error" else "qgemm_kernel (Y = X Q_R)",
            "bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
            "frac": achieved / peak_tf if peak_tf else None, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": "FP64 DMMA (mma.sync m8n8k4 f64) peak: max of the live probe (qcur_fp64_peak_tflops) and "
                           "the committed sustained microbenchmark (profiles/r01_fp64_peak_sustained.jsonl); "
                           "MEASURED_PEAKS.json has no FP64 figure", "peak_live": peak_live,
            "algorithmic_flop_per_launch": dom_flop, "avg_launch_ms": dom_ms,
        }
    t_roof = max(counts["flop"] / (peak_tf * 1e12), counts["bytes"] / ((hbm_peak or 6544.3) * 1e9))
    step_roof = {"note": "the reference's algorithmic flops at the FP64 DMMA peak (and its bytes at HBM peak); "
                         "the INT8 engine computes the big products exactly on the int8 tensor cores, so it can "
                         "run below this FP64 bound (frac > 1)",
                 "flop": counts["flop"], "bytes": counts["bytes"], "t_roofline_ms": t_roof * 1e3,
                 "frac": (t_roof * 1e3) / (ms_step / batch)}
    extra_phase = {}
    if "length" in per_approx:
        extra_phase["length_GBps"] = counts["length_bytes"] / (per_approx["length"] * 1e-3) / 1e9
        extra_phase["length_frac_hbm"] = extra_phase["length_GBps"] / (hbm_peak or 6544.3)
    if "gather" in per_approx:
        extra_phase["gather_GBps"] = counts["gather_bytes"] / (per_approx["gather"] * 1e-3) / 1e9
    extra_phase["gemm_xq_TFps"] = counts["gemm_xq_flop"] / (per_approx.get("gemm_xq", float("nan")) * 1e-3) / 1e12
    extra_phase["error_TFps"] = counts["error_flop"] / (per_approx.get("error", float("nan")) * 1e-3) / 1e12
    gp = graph_phases if isinstance(graph_phases, dict) else {}
    if isinstance(gp.get("length"), float) and gp["length"] > 0:  # the same rates as the graph replays run them
        extra_phase["length_GBps_in_graph"] = counts["length_bytes"] / (gp["length"] * 1e-3) / 1e9
        extra_phase["length_frac_hbm_in_graph"] = extra_phase["length_GBps_in_graph"] / (hbm_peak or 6544.3)
    if isinstance(gp.get("gather"), float) and gp["gather"] > 0:
        extra_phase["gather_GBps_in_graph"] = counts["gather_bytes"] / (gp["gather"] * 1e-3) / 1e9

    # --- e2e through the public API with pinned host buffers ---
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    pinned = [torch.empty((m, n), dtype=torch.float64, pin_memory=True) for _ in range(4)]
    host_planes = [p.numpy() for p in pinned]
    dev.download_planes(xs[0], m, n, pinned_out=host_planes)
    xh = QMatrix._wrap(*host_planes)

    def e2e_step():
        drop_device_copy(xh)
        plan = make_plan(xh, cfg["strategy"], cfg["rank"], cfg["plan_seed"], num_rows=r, num_cols=c)
        f = qmcur(xh, plan)
        return cur_relative_error(xh, f)

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_err = e2e_step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    tt = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_s = float(tt.item())
    e2e = {
        "value": world * e2e_steps / e2e_s,
        "unit": "approx/s",
        "h2d_bytes_per_step": 32 * m * n + 8 * (m + n),
        "d2h_bytes_per_step": 8 * (m + n) + 32 * (m * c + c * r + r * n) + 8 * (c + r) + 16,
        "api": "make_plan + qmcur + cur_relative_error on a QMatrix with pinned host planes (device cache dropped "
               "every step)",
        "steps": e2e_steps,
        "rel_err": e2e_err,
    }
    # the same work through the throughput API (approx_stream): matrix k+1's H2D overlaps
    # matrix k's approximation; every step still uploads its 512 MB and reads back its result
    # (two device slots of X: skipped when they would not leave room for the pipeline, e.g. cfg5)
    total_mem = torch.cuda.get_device_properties(local).total_memory
    if batch == 1 and 2 * 32 * m * n <= 0.25 * total_mem:
        from paper_2402_19147_b200 import approx_stream

        nst = max(e2e_steps, 6)
        seeds = [cfg["plan_seed"]] * (nst + 2)
        list(approx_stream([xh] * 2, cfg["strategy"], cfg["rank"], seeds[:2], num_rows=r, num_cols=c))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        res_s = list(approx_stream([xh] * nst, cfg["strategy"], cfg["rank"], seeds[:nst], num_rows=r, num_cols=c))
        torch.cuda.synchronize()
        st_s = time.perf_counter() - t0
        tt = torch.tensor([st_s], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        st_s = float(tt.item())
        # headline e2e = the drop-in call a reference user makes (make_plan + qmcur +
        # cur_relative_error, factors returned to the host); the throughput API rides beside it
        e2e["approx_stream"] = {
            "value": world * nst / st_s, "unit": "approx/s", "steps": nst,
            "h2d_bytes_per_step": 32 * m * n, "d2h_bytes_per_step": 32 * c * r + 8 * (c + r) + 36,
            "api": f"approx_stream over pinned host matrices: each step uploads its {32 * m * n / 1e6:.0f} MB input "
                   "(H2D of the next overlapped with the current approximation) and reads back its indices, U and error",
            "rel_err": res_s[-1].rel_err,
        }

    # --- CPU baseline (rank 0, N = 1): the unmodified reference (baseline/_ref) on this host's
    # cores, one bounded step in a thread-capped subprocess; the oracle port on the GPU's own
    # input checks agreement ---
    cpu = None
    if cfg.get("no_cpu") and not args.no_cpu_baseline:
        cpu = {"value": None, "unit": "approx/s", "cores": cpu_threads(), "kind": "reference",
               "sample": "not run: the reference needs ~100 GB of host temporaries and hours for one 32768^2 "
                         "approximation"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O

        planes = tuple(np.array(p) for p in host_planes)
        # the GPU's error on the same matrix (xs[0]) and plan seed as the CPU sample (in a batch the
        # timed loop's last error belongs to another matrix)
        seed0 = cfg["plan_seed"] + mine[0]
        outs.run(xs[0], cfg["strategy"], seed0, psnr_scale, graph=False)
        rel_err0 = outs.rel_error()
        t0 = time.perf_counter()
        res = O.approx(planes, cfg["strategy"], cfg["rank"], seed0, c, r)
        cpu_s = time.perf_counter() - t0
        port = {"value": 1.0 / cpu_s, "unit": "approx/s", "cores": cpu_threads(), "kind": "port",
                "sample": f"1 full approximation of {args.config} (make_plan + qmcur + relative error) "
                          f"by oracle/oracle.py on the GPU's own input",
                "rel_err": res["rel_err"], "agrees_with_gpu_rel": abs(res["rel_err"] - rel_err0) / res["rel_err"]}
        ref = reference_subprocess(args.config, cfg, 1, 0, 60.0)
        if ref is not None:
            t_ref = sum(ref["times"])
            cpu = {"value": len(ref["times"]) * batch / t_ref, "unit": "approx/s", "cores": ref["cores"],
                   "kind": "reference",
                   "sample": f"{len(ref['times'])} step(s) of {batch} approximation(s) of {args.config} by the "
                             f"unmodified reference (baseline/_ref, public API, BLAS threads = {ref['cores']}) on "
                             f"the host-generated twin of the workload",
                   "rel_err": ref["rel_err"], "port": port}
        else:
            cpu = port

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "approx/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if batch > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: on-device Philox Gaussian quaternion factors, S = P Q^H on DMMA, Gaussian noise",
            "config": {"workload": workload_name(args.config, cfg), "m": m, "n": n, "c": c, "r": r,
                       "strategy": cfg["strategy"], "batch": batch,
                       "parallelism": ("single GPU" if world == 1 else
                                       (f"batch split by matrix over {world} GPUs" if batch > 1
                                        else f"replicas x{world}")),
                       "l2": f"inputs larger than L2 ({m * n * 32 / 1e6:.0f} MB per matrix); no flush"
                       if m * n * 32 > 126e6
                       else "input fits in L2; repeated on the same resident matrix",
                       "launch": ((f"one CUDA graph replay per step: qcur_approx_batched over this rank's "
                                   f"{len(mine)} matrices on {bt.lanes} lanes" if bt is not None else
                                   "one CUDA graph replay per approximation (captured from the same ABI call)")
                                  if use_graph else "direct stream launches"),
                       "inflight": len(lanes),
                       "inflight_note": "approximations in flight: independent resident inputs of this workload, "
                                        "one native context and stream each, steps round-robin over them; "
                                        "value_serial is the same loop with one in flight"},
            "value_serial": serial,
            "gpu_launches": launches, "rel_err": rel_err, "batch_results": batch_results,
            "psnr": (dict(zip(("u8_db", "float_peak1_db"), outs.psnr())) if psnr_scale else None),
            "roofline": roofline, "step_roofline": step_roof,
            "phases_ms_per_approx": per_approx, "phases_in_graph_ms_per_approx": graph_phases,
            "phase_rates": extra_phase,
            "clocks": sampler.summary(), "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
