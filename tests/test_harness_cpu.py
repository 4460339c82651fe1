"""Study-driver logic that needs no device (harness.py semantics)."""

import numpy as np
import pytest

from paper_1805_02144_b200.harness import (CSV_HEADER, ResultRow, _check, fit_order,
                                           rel_linf_error, write_csv)


def test_csv_schema(tmp_path):
    rows = [ResultRow("exprb42", 600.0, 1.5e-7, 0.25, 10, 700, 20)]
    p = tmp_path / "out.csv"
    write_csv(rows, p)
    lines = p.read_text().splitlines()
    assert lines[0] == CSV_HEADER == "scheme,dt,error_linf,cpu_seconds,steps,matvecs,substeps"
    assert lines[1].split(",")[0] == "exprb42" and len(lines[1].split(",")) == 7


def test_fit_order_slopes():
    dts = [0.4, 0.2, 0.1, 0.05]
    rows = [ResultRow("s", d, 3.0 * d ** 4, 0, 0, 0, 0) for d in dts]
    slope, flagged = fit_order(rows, 1e-12)
    assert slope == pytest.approx(4.0) and not flagged
    rows[-1].error_linf = 1e-14
    rows[-2].error_linf = 1e-14
    slope, flagged = fit_order(rows, 1e-12)
    assert slope is None and len(flagged) == 2


def test_dt_validation():
    with pytest.raises(ValueError):
        _check(("exprb42",), (1.0, 2.0))
    with pytest.raises(ValueError):
        _check(("nope",), (2.0, 1.0))
    assert _check(("epi3",), (2, 1)) == (2.0, 1.0)


def test_rel_linf_height_slice():
    u = np.array([0.0, 0.0, 1.0, 2.0])
    ref = np.array([5.0, 5.0, 1.0, 4.0])
    assert rel_linf_error(u, ref, slice(2, 4)) == pytest.approx(0.5)
