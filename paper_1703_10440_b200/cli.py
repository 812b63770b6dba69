"""Command-line front end: the reference's ``factor`` and ``bench``
subcommands on the B200 path (cli.py:88-166).

    python -m paper_1703_10440_b200 factor --a A.mtx --z Z.mtx --method mgs-ha-row [--out-q Q.mtx] [--out-r R.mtx] [--report]
    python -m paper_1703_10440_b200 bench --kind laplacian --m 1048576 --n-list 16,64 --out bench.csv

Exit codes as the reference: 0 success; 2 bad flags or malformed /
ill-shaped input; 3 factorization failure (breakdown or loss of positive
definiteness).  Each run echoes its resolved configuration to stderr; CSV
outputs carry the same line as a leading ``#`` comment.  The reference's
``sweep`` / ``check`` (the accuracy study) are out of scope.
"""

import argparse
import sys

from .exceptions import (
    AqrError,
    BreakdownError,
    DimensionError,
    NotPositiveDefiniteError,
    ParseError,
    UnsupportedFormatError,
)
from .gram_schmidt import SWEEP_METHODS, MethodId, factorize
from .metrics import loss_of_A_orthogonality, representation_error
from .mmio import read_matrix_market, write_matrix_market
from .operators import SpdOperator, as_matrix, as_operator
from .timing import BENCH_METHODS, run_bench

BENCH_COLUMNS = "kind,m,n,method,seconds,mv_count"
BACKEND = "b200"


def _fmt(value):
    if value is None:
        return ""
    if isinstance(value, float):
        return repr(value)
    return str(value)


def _echo(text):
    print(f"# aqr {text}", file=sys.stderr)


def _parse_methods(text, default):
    if text is None:
        return list(default)
    if text.strip().lower() == "all":
        return list(SWEEP_METHODS)
    return [MethodId.parse(part) for part in text.split(",") if part.strip()]


def cmd_factor(args):
    a_obj = read_matrix_market(args.a)
    z_obj = read_matrix_market(args.z)
    op = as_operator(a_obj)
    Z = z_obj.to_dense() if isinstance(z_obj, SpdOperator) else as_matrix(z_obj)
    method = MethodId.parse(args.method)
    _echo(f"factor a={args.a} z={args.z} method={method} backend={BACKEND}")
    try:
        result = factorize(Z, op, method)
    except (BreakdownError, NotPositiveDefiniteError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    if args.out_q:
        write_matrix_market(args.out_q, result.Q, comment=f"Q factor, method {method}")
    if args.out_r:
        write_matrix_market(args.out_r, result.R, comment=f"R factor, method {method}")
    if args.report:
        loss = loss_of_A_orthogonality(result.Q, op)
        rep_rel = representation_error(Z, result.Q, result.R)[1]
        print(f"{result.cost.mv_count},{result.cost.flops},{_fmt(loss)},{_fmt(rep_rel)}")
    return 0


def cmd_bench(args):
    n_list = [int(part) for part in args.n_list.split(",") if part.strip()]
    methods = _parse_methods(args.methods, BENCH_METHODS)
    config = (f"bench kind={args.kind} m={args.m} n_list={args.n_list} seed={args.seed} "
              f"methods={','.join(str(m) for m in methods)} backend={BACKEND} timer=perf_counter")
    _echo(config)
    records = run_bench(args.kind, args.m, n_list, args.seed, methods)
    with open(args.out, "w", encoding="ascii", newline="\n") as fh:
        fh.write(f"# aqr {config}\n")
        fh.write(BENCH_COLUMNS + "\n")
        for r in records:
            fh.write(f"{r.kind},{r.m},{r.n},{r.method},{_fmt(r.seconds)},{r.mv_count}\n")
    print(f"wrote {len(records)} records to {args.out}", file=sys.stderr)
    return 0


def build_parser():
    parser = argparse.ArgumentParser(prog="python -m paper_1703_10440_b200",
                                     description="A-orthogonal MGS QR on the B200 (arXiv 1703.10440)")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("factor", help="factor one instance from Matrix Market files")
    p.add_argument("--a", required=True, help="weight matrix A (.mtx, array or coordinate)")
    p.add_argument("--z", required=True, help="matrix Z to factor (.mtx)")
    p.add_argument("--method", required=True, help="method id: {mgs|cgs}-{naive|ha|hp}-{col|row} or cholqr")
    p.add_argument("--out-q", help="write Q here (Matrix Market array)")
    p.add_argument("--out-r", help="write R here (Matrix Market array)")
    p.add_argument("--report", action="store_true",
                   help="print one CSV line: mv_count,flops,loss_a_orth,rep_error_rel")
    p.set_defaults(func=cmd_factor)
    p = sub.add_parser("bench", help="wall-clock benchmark")
    p.add_argument("--kind", choices=("dense", "laplacian"), required=True)
    p.add_argument("--m", type=int, required=True)
    p.add_argument("--n-list", required=True, help="comma list of n values")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--methods", help="comma list of method ids (default: mgs trio + cholqr)")
    p.add_argument("--out", required=True, help="output CSV path")
    p.set_defaults(func=cmd_bench)
    return parser


def main(argv=None):
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        return args.func(args)
    except (ParseError, UnsupportedFormatError, DimensionError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except AqrError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3


def entry():
    sys.exit(main())
