"""Report and trace serialisation.

The reference package never implemented its CLI; its specification fixes the
file formats (`SPEC.md:644-654` of the reference): JSON for structured
reports with a ``"schema": 1`` field, CSV for arrays and the iteration trace
(locale-independent, ``.`` decimal, ``\\n`` rows), floats written with 17
significant digits so that they read back bit-exactly.  Non-finite floats
(e.g. the NaN criterion fields of a pure-EG trace) are written as ``nan``,
``inf`` and ``-inf`` — JSON strings in a report, bare tokens in a CSV.

Host-side only: nothing here touches the device.
"""

from __future__ import annotations

import dataclasses
import io
import json
import math
from typing import Any

import numpy as np

from paper_2310_14087_b200.solver import IterationRecord, SolverReport

SCHEMA = 1
_FIELDS = [f.name for f in dataclasses.fields(IterationRecord)]


def fmt_float(x: float) -> str:
    """17 significant digits (round-trip exact); ``nan`` / ``inf`` / ``-inf`` for non-finite values."""
    x = float(x)
    if math.isnan(x):
        return "nan"
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    s = format(x, ".17g")
    return s if any(c in s for c in ".e") else s + ".0"  # stays a float (and keeps −0.0) when parsed


def parse_float(s: str) -> float:
    return float(s)  # float() accepts nan / inf / -inf and every %.17g string


def _json_value(v: Any) -> str:
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        s = fmt_float(v)
        return s if math.isfinite(float(v)) else json.dumps(s)
    if v is None:
        return "null"
    if isinstance(v, str):
        return json.dumps(v)
    if isinstance(v, np.ndarray):
        return _json_value(v.tolist())
    if isinstance(v, (list, tuple)):
        return "[" + ",".join(_json_value(x) for x in v) + "]"
    if isinstance(v, dict):
        return "{" + ",".join(json.dumps(str(k)) + ":" + _json_value(x) for k, x in v.items()) + "}"
    raise TypeError(f"cannot serialise {type(v).__name__}")


def report_dict(rep: SolverReport, include_x: bool = False) -> dict:
    """The structured report: scalars, γ̂ (and optionally X̂) and the trace as a list of records."""
    d = {
        "schema": SCHEMA,
        "termination": rep.termination,
        "iterations": rep.iterations,
        "residual_norm": float(rep.residual_norm),
        "ot_estimate": None if rep.ot_estimate is None else float(rep.ot_estimate),
        "total_ms": float(rep.total_ms),
        "gamma_hat": np.asarray(rep.gamma_hat, dtype=np.float64),
        "trace": [dataclasses.asdict(r) for r in rep.trace],
    }
    if include_x and rep.x_hat is not None:
        d["x_hat"] = np.asarray(rep.x_hat, dtype=np.float64)
    return d


def dumps_report(rep: SolverReport, include_x: bool = False) -> str:
    return _json_value(report_dict(rep, include_x)) + "\n"


def _restore(v: Any) -> Any:
    if isinstance(v, str) and v in ("nan", "inf", "-inf"):
        return float(v)
    if isinstance(v, list):
        return [_restore(x) for x in v]
    if isinstance(v, dict):
        return {k: _restore(x) for k, x in v.items()}
    return v


def loads_report(text: str) -> SolverReport:
    """Inverse of :func:`dumps_report` (bit-exact for every float)."""
    d = _restore(json.loads(text))
    if d.get("schema") != SCHEMA:
        raise ValueError(f"unsupported report schema {d.get('schema')!r}")
    trace = [IterationRecord(**r) for r in d["trace"]]
    x = np.asarray(d["x_hat"], dtype=np.float64) if "x_hat" in d else None
    return SolverReport(gamma_hat=np.asarray(d["gamma_hat"], dtype=np.float64), x_hat=x,
                        ot_estimate=d["ot_estimate"], residual_norm=d["residual_norm"],
                        termination=d["termination"], trace=trace, total_ms=d["total_ms"])


def write_report_json(rep: SolverReport, path: str, include_x: bool = False) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write(dumps_report(rep, include_x))


def read_report_json(path: str) -> SolverReport:
    with open(path, encoding="utf-8") as f:
        return loads_report(f.read())


def _cell(v: Any) -> str:
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return fmt_float(v)
    return str(v)


def dumps_trace_csv(trace: list[IterationRecord]) -> str:
    out = io.StringIO()
    out.write(",".join(_FIELDS) + "\n")
    for r in trace:
        out.write(",".join(_cell(getattr(r, k)) for k in _FIELDS) + "\n")
    return out.getvalue()


def loads_trace_csv(text: str) -> list[IterationRecord]:
    lines = [ln for ln in text.split("\n") if ln]
    if not lines or lines[0].split(",") != _FIELDS:
        raise ValueError("not an iteration-trace CSV (header mismatch)")
    types = {f.name: f.type for f in dataclasses.fields(IterationRecord)}
    recs = []
    for ln in lines[1:]:
        vals = ln.split(",")
        kw = {}
        for k, s in zip(_FIELDS, vals):
            t = types[k]
            if t in (int, "int"):
                kw[k] = int(s)
            elif t in (bool, "bool"):
                kw[k] = s == "true"
            elif t in (str, "str"):
                kw[k] = s
            else:
                kw[k] = parse_float(s)
        recs.append(IterationRecord(**kw))
    return recs


def write_trace_csv(trace: list[IterationRecord], path: str) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write(dumps_trace_csv(trace))


def read_trace_csv(path: str) -> list[IterationRecord]:
    with open(path, encoding="utf-8") as f:
        return loads_trace_csv(f.read())


def dumps_array_csv(a) -> str:
    """A vector as one value per row, a matrix as one row per line (17 significant digits)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        return "".join(fmt_float(x) + "\n" for x in a)
    if a.ndim == 2:
        return "".join(",".join(fmt_float(x) for x in row) + "\n" for row in a)
    raise ValueError("arrays of rank 1 or 2 only")


def loads_array_csv(text: str) -> np.ndarray:
    rows = [ln.split(",") for ln in text.split("\n") if ln]
    if rows and all(len(r) == 1 for r in rows):
        return np.array([parse_float(r[0]) for r in rows], dtype=np.float64)
    return np.array([[parse_float(x) for x in r] for r in rows], dtype=np.float64)
