"""Report / trace serialisation: bit-exact round trips, CPU only."""

import math

import numpy as np
import pytest

from paper_2310_14087_b200 import report as R
from paper_2310_14087_b200.solver import IterationRecord, SolverReport


def _same(a, b):
    if isinstance(a, float) and isinstance(b, float):
        return (math.isnan(a) and math.isnan(b)) or a == b and math.copysign(1, a) == math.copysign(1, b)
    return a == b


def _synthetic(seed=0, n=7, iters=5):
    rng = np.random.default_rng(seed)
    trace = []
    for k in range(iters):
        vals = [float(v) for v in rng.standard_normal(12) * 10.0 ** rng.integers(-300, 300, 12)]
        trace.append(IterationRecord(k, *vals[:3], "ssn" if k % 2 else "eg", *vals[3:5], int(rng.integers(0, 60)),
                                     bool(k % 2), float("nan") if k == 0 else vals[5],
                                     float("inf") if k == 1 else vals[6], *vals[7:12], int(rng.integers(0, n)),
                                     int(rng.integers(1, 4))))
    g = rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20, n)
    g[0] = -0.0
    x = rng.standard_normal((n, n))
    return SolverReport(gamma_hat=g, x_hat=x @ x.T, ot_estimate=float(rng.standard_normal()), residual_norm=1e-7,
                        termination="max_iter", trace=trace, total_ms=123.456)


def test_float_format_is_17_digits_and_round_trips():
    rng = np.random.default_rng(1)
    for x in np.concatenate([rng.standard_normal(200) * 10.0 ** rng.integers(-308, 308, 200),
                             [5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 0.1, -0.0]]):
        s = R.fmt_float(x)
        assert R.parse_float(s) == x and math.copysign(1, R.parse_float(s)) == math.copysign(1, x)
    assert R.fmt_float(0.1) == "0.10000000000000001"
    assert [R.fmt_float(v) for v in (float("nan"), float("inf"), -float("inf"))] == ["nan", "inf", "-inf"]


@pytest.mark.parametrize("include_x", [False, True])
def test_report_json_round_trip_is_exact(tmp_path, include_x):
    rep = _synthetic()
    p = tmp_path / "report.json"
    R.write_report_json(rep, str(p), include_x=include_x)
    text = p.read_text()
    assert '"schema":1' in text and "NaN" not in text and "Infinity" not in text  # strict JSON
    back = R.read_report_json(str(p))
    assert np.array_equal(back.gamma_hat, rep.gamma_hat) and math.copysign(1, back.gamma_hat[0]) < 0
    assert (back.x_hat is not None) == include_x
    if include_x:
        assert np.array_equal(back.x_hat, rep.x_hat)
    assert (back.termination, back.iterations, back.residual_norm, back.ot_estimate, back.total_ms) == \
        (rep.termination, rep.iterations, rep.residual_norm, rep.ot_estimate, rep.total_ms)
    for a, b in zip(back.trace, rep.trace):
        for k in R._FIELDS:
            assert _same(getattr(a, k), getattr(b, k)), k


def test_trace_csv_round_trip_is_exact(tmp_path):
    rep = _synthetic(seed=3, iters=9)
    p = tmp_path / "trace.csv"
    R.write_trace_csv(rep.trace, str(p))
    raw = p.read_bytes()
    assert b"\r" not in raw and raw.startswith(b"iteration,res_accepted,res_ssn,res_eg,accepted")
    back = R.read_trace_csv(str(p))
    assert len(back) == len(rep.trace)
    for a, b in zip(back, rep.trace):
        for k in R._FIELDS:
            assert type(getattr(a, k)) is type(getattr(b, k)), k
            assert _same(getattr(a, k), getattr(b, k)), k


def test_array_csv_round_trip_is_exact():
    rng = np.random.default_rng(4)
    v = rng.standard_normal(11) * 1e-200
    m = rng.standard_normal((5, 3)) * 1e200
    assert np.array_equal(R.loads_array_csv(R.dumps_array_csv(v)), v)
    assert np.array_equal(R.loads_array_csv(R.dumps_array_csv(m)), m)
    with pytest.raises(ValueError):
        R.dumps_array_csv(np.zeros((2, 2, 2)))


def test_rejects_foreign_files():
    with pytest.raises(ValueError):
        R.loads_report('{"schema": 2}')
    with pytest.raises(ValueError):
        R.loads_trace_csv("a,b,c\n1,2,3\n")
