"""Command line of the B200 path: ``factor`` and ``bench``.

    python -m paper_1703_10440_b200 factor --a A.mtx --z Z.mtx --method mgs-ha-row [--out-q Q.mtx] [--out-r R.mtx] [--report]
    python -m paper_1703_10440_b200 bench --kind laplacian --m 1048576 --n-list 16,64 --out bench.csv

Flags, CSV layout and exit statuses are those of the reference's
subcommands of the same names (/root/reference/pkg/src/aqr/cli.py:88-166):
0 on success, 2 for bad flags or unreadable / ill-shaped input, 3 when the
factorization itself fails (breakdown, Cholesky pivot).  The resolved
configuration is logged to stderr and repeated as the first (``#``) line of
a CSV output.  The reference's ``sweep`` / ``check`` (its accuracy study)
are out of scope.
"""

import argparse
import sys

from . import exceptions as E
from .gram_schmidt import SWEEP_METHODS, MethodId, factorize
from .metrics import loss_of_A_orthogonality, representation_error
from .mmio import read_matrix_market, write_matrix_market
from .operators import SpdOperator, as_matrix, as_operator
from .timing import BENCH_METHODS, run_bench

BACKEND = "b200"
EXIT_OK, EXIT_USAGE, EXIT_FAILED = 0, 2, 3
BENCH_FIELDS = ("kind", "m", "n", "method", "seconds", "mv_count")
BENCH_COLUMNS = ",".join(BENCH_FIELDS)

# input problems -> exit 2; failures of the factorization itself -> exit 3
_USAGE_ERRORS = (E.ParseError, E.UnsupportedFormatError, E.DimensionError, ValueError, OSError)
_RUN_ERRORS = (E.BreakdownError, E.NotPositiveDefiniteError)


def _log(line):
    sys.stderr.write(f"# aqr {line}\n")


def _cell(v):
    """CSV cell: floats round-trip exactly (repr), None is empty."""
    return "" if v is None else (repr(v) if isinstance(v, float) else str(v))


def _methods(spec, fallback):
    if spec is None:
        return list(fallback)
    if spec.strip().lower() == "all":
        return list(SWEEP_METHODS)
    return [MethodId.parse(tok) for tok in spec.split(",") if tok.strip()]


class FactorCommand:
    name = "factor"
    help = "factor one instance read from Matrix Market files"

    def add_arguments(self, p):
        p.add_argument("--a", required=True, help="weight matrix A (.mtx, array or coordinate)")
        p.add_argument("--z", required=True, help="matrix Z to factor (.mtx)")
        p.add_argument("--method", required=True, help="{mgs|cgs}-{naive|ha|hp}-{col|row} or cholqr")
        p.add_argument("--out-q", help="write Q here (Matrix Market array)")
        p.add_argument("--out-r", help="write R here (Matrix Market array)")
        p.add_argument("--report", action="store_true",
                       help="print one CSV line: mv_count,flops,loss_a_orth,rep_error_rel")

    def run(self, ns):
        weight, block = read_matrix_market(ns.a), read_matrix_market(ns.z)
        op = as_operator(weight)
        Z = block.to_dense() if isinstance(block, SpdOperator) else as_matrix(block)
        method = MethodId.parse(ns.method)
        _log(f"factor a={ns.a} z={ns.z} method={method} backend={BACKEND}")
        try:
            res = factorize(Z, op, method)
        except _RUN_ERRORS as exc:
            sys.stderr.write(f"error: {exc}\n")
            return EXIT_FAILED
        for path, factor, label in ((ns.out_q, res.Q, "Q"), (ns.out_r, res.R, "R")):
            if path:
                write_matrix_market(path, factor, comment=f"{label} factor, method {method}")
        if ns.report:
            cells = (res.cost.mv_count, res.cost.flops, loss_of_A_orthogonality(res.Q, op),
                     representation_error(Z, res.Q, res.R)[1])
            print(",".join(_cell(c) for c in cells))
        return EXIT_OK


class BenchCommand:
    name = "bench"
    help = "wall-clock benchmark of the methods over a list of n"

    def add_arguments(self, p):
        p.add_argument("--kind", choices=("dense", "laplacian"), required=True)
        p.add_argument("--m", type=int, required=True)
        p.add_argument("--n-list", required=True, help="comma list of n values")
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--methods", help="comma list of method ids (default: mgs trio + cholqr)")
        p.add_argument("--out", required=True, help="output CSV path")

    def run(self, ns):
        ns_list = [int(tok) for tok in ns.n_list.split(",") if tok.strip()]
        methods = _methods(ns.methods, BENCH_METHODS)
        header = (f"bench kind={ns.kind} m={ns.m} n_list={ns.n_list} seed={ns.seed} "
                  f"methods={','.join(map(str, methods))} backend={BACKEND} timer=perf_counter")
        _log(header)
        recs = run_bench(ns.kind, ns.m, ns_list, ns.seed, methods)
        lines = [f"# aqr {header}", BENCH_COLUMNS]
        lines += [",".join(_cell(getattr(r, f)) for f in BENCH_FIELDS) for r in recs]
        with open(ns.out, "w", encoding="ascii", newline="\n") as fh:
            fh.write("\n".join(lines) + "\n")
        sys.stderr.write(f"wrote {len(recs)} records to {ns.out}\n")
        return EXIT_OK


COMMANDS = (FactorCommand(), BenchCommand())


def build_parser():
    parser = argparse.ArgumentParser(prog="python -m paper_1703_10440_b200",
                                     description="A-orthogonal MGS QR on the B200 (arXiv 1703.10440)")
    sub = parser.add_subparsers(dest="command", required=True)
    for cmd in COMMANDS:
        p = sub.add_parser(cmd.name, help=cmd.help)
        cmd.add_arguments(p)
        p.set_defaults(command_obj=cmd)
    return parser


def main(argv=None):
    ns = build_parser().parse_args(argv)
    try:
        return ns.command_obj.run(ns)
    except _USAGE_ERRORS as exc:
        sys.stderr.write(f"error: {exc}\n")
        return EXIT_USAGE
    except E.AqrError as exc:
        sys.stderr.write(f"error: {exc}\n")
        return EXIT_FAILED


def entry():
    sys.exit(main())
