"""The reference's ``factor`` / ``bench`` command line on the B200 path
(reference cli.py:88-166 and test_cli.py)."""

import numpy as np
import pytest

from paper_1703_10440_b200 import cli
from paper_1703_10440_b200.mmio import read_matrix_market, write_matrix_market


def test_bad_flags_and_bad_input_exit_2(tmp_path, capsys):
    with pytest.raises(SystemExit) as info:
        cli.main(["factor", "--a", "x.mtx"])
    assert info.value.code == 2
    bad = tmp_path / "bad.mtx"
    bad.write_text("not a matrix market file\n")
    assert cli.main(["factor", "--a", str(bad), "--z", str(bad), "--method", "mgs-ha-row"]) == 2
    assert "line 1" in capsys.readouterr().err
    assert cli.main(["factor", "--a", str(tmp_path / "missing.mtx"), "--z", str(bad), "--method", "mgs-ha-row"]) == 2


@pytest.mark.gpu
def test_factor_writes_factors_and_report(tmp_path, capsys):
    from paper_1703_10440_b200 import factorize, laplacian_spd

    op = laplacian_spd(12, 10)
    Z = np.asfortranarray(np.random.default_rng(1).standard_normal((120, 6)))
    a, z, q, r = (tmp_path / f for f in ("a.mtx", "z.mtx", "q.mtx", "r.mtx"))
    write_matrix_market(a, op)
    write_matrix_market(z, Z)
    rc = cli.main(["factor", "--a", str(a), "--z", str(z), "--method", "mgs-hp-row",
                   "--out-q", str(q), "--out-r", str(r), "--report"])
    assert rc == 0
    ref = factorize(Z, laplacian_spd(12, 10), "mgs-hp-row")
    assert np.array_equal(read_matrix_market(q), ref.Q) and np.array_equal(read_matrix_market(r), ref.R)
    out = capsys.readouterr()
    mv, flops, loss, rep = out.out.strip().split(",")
    assert int(mv) == 6 and int(flops) == ref.cost.flops and float(loss) < 1e-13 and float(rep) < 1e-15
    assert "backend=b200" in out.err


@pytest.mark.gpu
def test_factor_breakdown_exit_3(tmp_path):
    a, z = tmp_path / "a.mtx", tmp_path / "z.mtx"
    write_matrix_market(a, np.eye(3))
    write_matrix_market(z, np.array([[1.0, 2.0], [0.0, 0.0], [0.0, 0.0]]))
    assert cli.main(["factor", "--a", str(a), "--z", str(z), "--method", "mgs-ha-col"]) == 3


@pytest.mark.gpu
def test_bench_csv(tmp_path):
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--kind", "laplacian", "--m", "400", "--n-list", "4,8", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0].startswith("# aqr bench kind=laplacian") and lines[1] == cli.BENCH_COLUMNS
    rows = [ln.split(",") for ln in lines[2:]]
    assert len(rows) == 2 * 4 and {r[3] for r in rows} == {"mgs-naive-col", "mgs-ha-col", "mgs-hp-col", "cholqr"}
    assert all(float(r[4]) > 0 for r in rows)
    assert cli.main(["bench", "--kind", "dense", "--m", "64", "--n-list", "5", "--methods", "mgs-ha-row",
                     "--out", str(out)]) == 0
