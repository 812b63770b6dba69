"""Every kernel variant kept behind an experiment knob computes the same bits.

The knobs exist only in the experiments build (libaqr_b200_exp.so,
-DAQR_EXPERIMENTS; the shipped libaqr_b200.so compiles them to their
defaults) and are read once per process, so each variant runs in a
subprocess on the experiments build and its factors are compared bitwise
with the shipped library's: the HP column loop's two-column trailing pass, the
unpipelined SpMV step, the windowed trailing passes' write-back period
(1 = the eager schedule: every pass rewrites the trailing block) and the
HP X catch-up period (0 = x formed from all finished p columns), the
separate R-row reduction launch, launches
without programmatic dependent launch, the materialized copy of Z, the
column-oriented loop for the col methods (by default they run the
row-oriented step schedule -- for HP that is also the eagerly updated X
against the shipped lazy x), and the per-step catch-up launches of the
host-input pipeline; the long-row (27-point) HA step with the deferred
update fused into the SpMV gathers instead of a separate pass; the plain CSR
kernels instead of the banded view of the stencil operators, and the banded
view's gather kernels instead of its shared-memory staged tiles.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {repo!r})
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems
ip, ix, dv = problems.laplacian5(700, 460, 1e-2)   # m = 322,000: the 2048-row tile path
m, n = 700 * 460, 20   # > 2 trailing windows and X catch-ups
Z = problems.rng(9, 7).standard_normal((n, m)).T
Zd = torch.from_numpy(np.ascontiguousarray(Z.T)).cuda().t()
op = aqr.CsrSpdOperator(ip, ix, dv)
out = {{}}
for meth in ("mgs-ha-row", "mgs-hp-row", "cgs-ha-row", "cgs-hp-row", "mgs-naive-row", "mgs-hp-col",
             "mgs-ha-col", "cgs-naive-col"):
    r = aqr.factorize(Zd, op, meth)
    out[meth + "|Q"] = r.Q.cpu().numpy()
    out[meth + "|R"] = r.R.cpu().numpy()
s27 = problems.stencil27_device(70, 1e-2, "cuda")  # long rows (27-point), 343,000 rows
op27 = aqr.CsrSpdOperator(*s27)
Z27 = torch.from_numpy(problems.rng(9, 8).standard_normal((10, 70 ** 3))).cuda().t()
for meth in ("mgs-ha-row", "cgs-ha-row", "mgs-hp-row"):
    r = aqr.factorize(Z27, op27, meth)
    out["st27|" + meth + "|Q"] = r.Q.cpu().numpy()
    out["st27|" + meth + "|R"] = r.R.cpu().numpy()
import os
os.environ["AQR_CHUNK_COLS"] = "3"  # host input: the chunked pipeline and its catch-up
Zn = np.asfortranarray(Z)
for meth in ("mgs-ha-row", "cgs-ha-row", "mgs-hp-row", "mgs-naive-col"):
    r = aqr.factorize(Zn, op, meth)
    out[meth + "|Qh"] = r.Q
    out[meth + "|Rh"] = r.R
np.savez({path!r}, **out)
"""


EXP_LIB = os.path.join(REPO, "paper_1703_10440_b200", "libaqr_b200_exp.so")


def _run(env_extra, path, lib=None):
    env = dict(os.environ)
    env.update(env_extra)
    env.pop("AQR_LIB_PATH", None)
    if lib:
        env["AQR_LIB_PATH"] = lib
    code = SCRIPT.format(repo=REPO, path=str(path))
    subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=600)
    return np.load(path)


@pytest.fixture(scope="module")
def default_factors(tmp_path_factory):
    return _run({}, tmp_path_factory.mktemp("v") / "default.npz")


@pytest.mark.parametrize("knobs", [
    {},
    {"AQR_TRAIL_WIN": "1"},
    {"AQR_TRAIL_WIN": "2"},
    {"AQR_TRAIL_WIN": "8"},
    {"AQR_X_WIN": "0"},
    {"AQR_X_WIN": "3"},
    {"AQR_SPMM_SG": "0"},
    {"AQR_XC_ROWS": "4"},
    {"AQR_XC_STREAM": "0"},
    {"AQR_SPLIT_LONG": "0"},
    {"AQR_BAND": "0"},
    {"AQR_BAND_STAGE": "0"},
    {"AQR_BAND": "0", "AQR_SPLIT_LONG": "0"},
    {"AQR_PIPE_MERGE": "0"},
    {"AQR_TRAIL_VARIANT": "6"},
    {"AQR_LDG_REVERSE": "0"},
    {"AQR_TRAIL_CTAS": "8"},
    {"AQR_PLAIN_PF": "0"},
    {"AQR_CATCHUP": "2"},
    {"AQR_PIPE_SCHED": "2"},
    {"AQR_SPMV_VARIANT": "3"},
    {"AQR_DEFER": "0"},
    {"AQR_PDL": "0"},
    {"AQR_DIRECT": "0"},
    {"AQR_COL_SCHEDULE": "1"},
    {"AQR_CATCHUP": "0"},
])
def test_variant_bitwise_equal_default(default_factors, knobs, tmp_path):
    got = _run(knobs, tmp_path / "variant.npz", lib=EXP_LIB)
    for key in default_factors.files:
        assert np.array_equal(got[key], default_factors[key]), (knobs, key)


def test_shipped_library_ignores_knobs(default_factors, tmp_path):
    """A stray experiment variable does not change the shipped library's schedule."""
    got = _run({"AQR_COL_SCHEDULE": "1", "AQR_DEFER": "0", "AQR_TRAIL_WIN": "1"}, tmp_path / "s.npz")
    for key in default_factors.files:
        assert np.array_equal(got[key], default_factors[key]), key
