"""Parity metrics and calibrated tolerances (test infrastructure).

The B200 kernels reproduce every elementwise operation and every operator
product of the reference bit for bit; only the dot-product reductions are
reordered (deterministic tree instead of a sequential chain).  The tolerance
for a case is therefore calibrated on the case itself: TOL_FACTOR times the
spread between the oracle with sequential dots (the reference) and the
oracle with pairwise dots (oracle.pairwise_dots), floored at FLOOR.
"""

import numpy as np

from oracle import oracle as O

TOL_FACTOR = 100.0
FLOOR = 1e-13
Q_COLUMN_FLOOR = 1e-3


def _np(a):
    return np.asarray(a.cpu() if hasattr(a, "cpu") else a)


def factor_errors(Q, R, Qref, Rref):
    """(Q error with column-norm floor, max|dR| / max|R|)."""
    Q, R, Qref, Rref = map(_np, (Q, R, Qref, Rref))
    colmax = np.abs(Qref).max(axis=0, keepdims=True)
    den = np.maximum(np.abs(Qref), Q_COLUMN_FLOOR * colmax)
    den = np.where(den > 0, den, 1.0)
    eq = float(np.max(np.abs(Q - Qref) / den))
    er = float(np.max(np.abs(R - Rref)) / max(float(np.max(np.abs(Rref))), 1e-300))
    return eq, er


def spread(Z, spec, method):
    seq = O.gs_factor(Z, spec, method)
    with O.pairwise_dots():
        pw = O.gs_factor(Z, spec, method)
    return factor_errors(pw.Q, pw.R, seq.Q, seq.R)


def tolerance(Z, spec, method):
    sq, sr = spread(Z, spec, method)
    return max(TOL_FACTOR * sq, FLOOR), max(TOL_FACTOR * sr, FLOOR)


def calibrated(Z, spec, methods, threads=None):
    """{method: (oracle result, q tolerance, r tolerance)} for one input.

    Runs the oracle with sequential dots (the reference) and with pairwise
    dots (the calibration) for every method concurrently on host threads
    (the C oracle releases the GIL; the dot mode is per thread)."""
    from concurrent.futures import ThreadPoolExecutor

    def seq(meth):
        return O.gs_factor(Z, spec, meth)

    def pw(meth):
        with O.pairwise_dots():
            return O.gs_factor(Z, spec, meth)

    jobs = [(meth, fn) for meth in methods for fn in (seq, pw)]
    with ThreadPoolExecutor(threads or len(jobs)) as ex:
        futs = {(meth, fn.__name__): ex.submit(fn, meth) for meth, fn in jobs}
    out = {}
    for meth in methods:
        s, p = futs[(meth, "seq")].result(), futs[(meth, "pw")].result()
        sq, sr = factor_errors(p.Q, p.R, s.Q, s.R)
        out[meth] = (s, max(TOL_FACTOR * sq, FLOOR), max(TOL_FACTOR * sr, FLOOR))
    return out
