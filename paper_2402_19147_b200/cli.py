"""Command-line front end for the QMCUR path: ``approx`` (cli.py:169-189).

    python -m paper_2402_19147_b200.cli approx INPUT.qmat --rank K [--strategy length|uniform]
                                            [--seed S] [--out DIR] [--time] [--verbose]

Same arguments, outputs (C.qmat, U.qmat, R.qmat, reconstruction.qmat and
metrics.csv with rel_err_fro, err_spec, time_s), seed derivation
(derive_seed(seed, "approx-draw")) and exit codes (0; 2 on QcurError / OSError)
as the reference's ``qcur approx``; every output is byte-reproducible run to run.
The other reference subcommands (image compression/inpainting, experiment
sweeps) are outside the accelerated path.
"""
from __future__ import annotations

import argparse
import logging
import sys
import time
from pathlib import Path

from .completion import derive_seed
from .cur import cur_reconstruct, make_plan, qmcur
from .errors import QcurError
from .linalg import spectral_norm
from .quat import qmat_frobenius_norm, read_qmat, write_qmat

__all__ = ["main", "cmd_approx"]


def _fmt(value: float) -> str:
    return format(float(value), ".17g")


def cmd_approx(args) -> int:
    x = read_qmat(args.input)
    plan = make_plan(x, args.strategy, args.rank, derive_seed(args.seed, "approx-draw"))
    if args.time:
        start = time.perf_counter()
        factors = qmcur(x, plan)
        elapsed = time.perf_counter() - start
    else:
        factors, elapsed = qmcur(x, plan), 0.0
    recon = cur_reconstruct(factors)
    diff = x - recon
    rel_err = qmat_frobenius_norm(diff) / qmat_frobenius_norm(x)
    err_spec = spectral_norm(diff)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    write_qmat(factors.c, out / "C.qmat")
    write_qmat(factors.u, out / "U.qmat")
    write_qmat(factors.r, out / "R.qmat")
    write_qmat(recon, out / "reconstruction.qmat")
    with open(out / "metrics.csv", "w", encoding="ascii", newline="") as fh:
        fh.write(f"rel_err_fro,err_spec,time_s\n{_fmt(rel_err)},{_fmt(err_spec)},{_fmt(elapsed)}\n")
    print(f"approx: rank {args.rank}, rel_err_fro={rel_err:.3e}; wrote {out}")
    return 0


def _build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="qcur-b200", description="Sampled quaternion CUR on the B200.")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("approx", help="factor a .qmat file and write C/U/R")
    p.add_argument("input", help="input .qmat file")
    p.add_argument("--rank", type=int, required=True)
    p.add_argument("--strategy", choices=("length", "uniform"), default="length")
    p.add_argument("--seed", type=int, default=0, help="master seed for all randomness")
    p.add_argument("--out", default=".", help="output directory (created if absent)")
    p.add_argument("--verbose", action="store_true", help="log per-step progress")
    p.add_argument("--time", action="store_true", help="measure wall time (makes CSV outputs nondeterministic)")
    return parser


def main(argv=None) -> int:
    args = _build_parser().parse_args(argv)
    logging.basicConfig(level=logging.DEBUG if args.verbose else logging.WARNING,
                        format="%(levelname)s %(name)s: %(message)s")
    try:
        return {"approx": cmd_approx}[args.command](args)
    except (QcurError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
