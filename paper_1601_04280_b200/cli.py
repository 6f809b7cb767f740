"""Command line: ``python -m paper_1601_04280_b200 decompose IN.mtx --r R``
(reference: cli.py:75-84, 87-104, 188-208 — the ``decompose`` subcommand;
the experiment-harness subcommands ``gen``/``run``/``cost`` are outside the
B200 path).  Writes P.mtx, Q.mtx (size x 1 arrays of exact float indices),
L.mtx and U.mtx to --out-dir and prints the reconstruction error.  Exit
codes as the reference: 0 success, 1 configuration/usage error, 2 numerical
failure.
"""

from __future__ import annotations

import argparse
import logging
import os
import sys

import numpy as np

from .errors import (DecompositionError, MatrixMarketError, ParameterError, ShapeError,
                     SingularMatrixError)

EXIT_OK = 0
EXIT_CONFIG = 1
EXIT_NUMERICAL = 2


class _UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # bad arguments are configuration errors (exit 1)
        raise _UsageError(message)


def build_parser():
    ap = _Parser(prog="python -m paper_1601_04280_b200",
                 description="B200 sparse randomized LU (arXiv 1601.04280)")
    sub = ap.add_subparsers(dest="command", required=True, parser_class=_Parser)
    dec = sub.add_parser("decompose", help="factor a Matrix Market file")
    dec.add_argument("input", help="input .mtx path")
    dec.add_argument("--r", type=int, required=True)
    dec.add_argument("--out-dir", default=".", help="directory for P/Q/L/U .mtx files")
    dec.add_argument("--seed", type=int, default=0)
    dec.add_argument("--mode", choices=("practical", "theoretical"), default="practical")
    dec.add_argument("--threads", type=int, default=None, help="host BLAS threads (parsing)")
    return ap


def main(argv=None) -> int:
    logging.basicConfig(format="%(levelname)s %(name)s: %(message)s")
    try:
        args = build_parser().parse_args(argv)
    except _UsageError as err:
        print(f"error: {err}", file=sys.stderr)
        return EXIT_CONFIG
    try:
        return _decompose(args)
    except (ParameterError, ShapeError, MatrixMarketError, OSError) as err:
        print(f"error: {err}", file=sys.stderr)
        return EXIT_CONFIG
    except (SingularMatrixError, DecompositionError) as err:
        print(f"numerical failure: {err}", file=sys.stderr)
        return EXIT_NUMERICAL


def _decompose(args) -> int:
    from .matrix import Matrix
    from .mmio import mm_read, mm_write, mm_write_host
    from .randlu import approximation_error, default_params, sparse_randomized_lu
    a = mm_read(args.input)
    params = default_params(args.r, a.rows, a.cols, field=a.field, seed=args.seed,
                            mode=args.mode)
    res = sparse_randomized_lu(a, params)
    os.makedirs(args.out_dir, exist_ok=True)
    mm_write_host(res.P.indices[:, None].astype(np.float64), os.path.join(args.out_dir, "P.mtx"))
    mm_write_host(res.Q.indices[:, None].astype(np.float64), os.path.join(args.out_dir, "Q.mtx"))
    mm_write(res.L, os.path.join(args.out_dir, "L.mtx"))
    mm_write(res.U, os.path.join(args.out_dir, "U.mtx"))
    err = approximation_error(a, res)
    fro = frobenius_norm(a)
    rel = err / fro if fro > 0 else 0.0
    print(f"decomposed {a.rows} x {a.cols} matrix at rank {params.r}: "
          f"|LU - PAQ|_F = {err:.6e} ({rel:.3e} relative), {res.elapsed['total']:.3f}s")
    return EXIT_OK


def frobenius_norm(a) -> float:
    """matrix.py frobenius_norm: sqrt of the sum of squares (fp64)."""
    import torch
    if a.is_sparse:
        return float(torch.linalg.vector_norm(a.raw[2].double()))
    return float(torch.linalg.vector_norm(a.raw.double()))


if __name__ == "__main__":
    sys.exit(main())
