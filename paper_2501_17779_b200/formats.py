"""Curve and result file formats (reference: proj/include/curvalign/io.hpp:10-33,
proj/src/io.cpp:44-151) — the data formats either side of the alignment path.

Host-side text handling (no GPU work). Same behaviour as the reference:
CSV is one "x,y" pair per line with an optional header, JSON is
``{"closed": true, "nodes": [[x, y], ...]}``; a closing duplicate node is
dropped on read; readers validate the curve (>= 4 finite nodes, curve.cpp:11-14);
CSV cells use 17 significant digits, JSON numbers the shortest round-trip
form with sorted keys (nlohmann::json::dump, the reference's writer).
Reader errors raise RuntimeError (the reference's std::runtime_error), except
the curve validation's ValueError (std::invalid_argument).
"""
from __future__ import annotations

import json
import math
import re

import numpy as np

__all__ = ["read_curve_csv", "write_curve_csv", "read_curve_json", "write_curve_json", "load_curve",
           "curve_to_csv", "curve_to_json", "alignment_to_json", "elastic_to_json", "matrix_to_csv"]


def _validate(c: np.ndarray) -> np.ndarray:  # validate_curve(c, 4) (curve.cpp:11-14)
    if c.shape[0] < 4:
        raise ValueError("curve: too few nodes")
    if not np.isfinite(c).all():
        raise ValueError("curve: non-finite node")
    return c


def _drop_closing_duplicate(nodes: list) -> list:  # io.cpp:28-33
    if len(nodes) >= 2 and nodes[0][0] == nodes[-1][0] and nodes[0][1] == nodes[-1][1]:
        nodes.pop()
    return nodes


_NUM = re.compile(r"\s*([+-]?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan))", re.IGNORECASE)


def _stod(t: str) -> float:
    """std::stod (strtod) acceptance: leading blanks skipped, the longest numeric
    prefix parsed, trailing characters ignored; no number, overflow or
    underflow (ERANGE) -> ValueError, as stod throws."""
    m = _NUM.match(t)
    if not m:
        raise ValueError(t)
    tok = m.group(1)
    v = float(tok)
    is_special = tok.lstrip("+-").lower().startswith(("inf", "nan"))
    if not is_special:
        digits_nonzero = any(ch in "123456789" for ch in tok.split("e")[0].split("E")[0])
        if math.isinf(v) or (digits_nonzero and abs(v) < 2.2250738585072014e-308):
            raise ValueError(t)
    return v


def _fmt17(v: float) -> str:  # ostream precision 17 (io.cpp:35-40)
    return format(v, ".17g")


def _jnum(v: float):
    return v if math.isfinite(v) else None


def read_curve_csv(path: str) -> np.ndarray:
    try:
        with open(path, "r", newline="") as f:
            text = f.read()
    except OSError as e:
        raise RuntimeError(f"cannot open file: {path}") from e
    nodes, header_allowed = [], True
    for line in text.split("\n"):
        if line in ("", "\r"):
            continue
        comma = line.find(",")
        if comma < 0 or comma + 1 == len(line):
            raise RuntimeError(f"malformed CSV line in {path}: {line}")
        try:
            x, y = _stod(line[:comma]), _stod(line[comma + 1:])
            ok = True
        except ValueError:
            ok = False
        header, header_allowed = (not ok and header_allowed), False
        if header:
            continue
        if not ok:
            raise RuntimeError(f"malformed CSV line in {path}: {line}")
        nodes.append((x, y))
    return _validate(np.array(_drop_closing_duplicate(nodes), dtype=np.float64).reshape(-1, 2))


def curve_to_csv(c) -> str:
    a = np.asarray(c, dtype=np.float64)
    return "x,y\n" + "".join(f"{_fmt17(x)},{_fmt17(y)}\n" for x, y in a)


def write_curve_csv(path: str, c) -> None:
    try:
        with open(path, "w", newline="") as f:
            f.write(curve_to_csv(c))
    except OSError as e:
        raise RuntimeError(f"cannot write file: {path}") from e


def read_curve_json(path: str) -> np.ndarray:
    try:
        with open(path, "r") as f:
            j = json.load(f)
    except OSError as e:
        raise RuntimeError(f"cannot open file: {path}") from e
    except json.JSONDecodeError as e:
        raise RuntimeError(f"JSON parse error in {path}: {e}") from e
    if not isinstance(j, dict) or not isinstance(j.get("nodes"), list):
        raise RuntimeError(f'curve JSON must contain a "nodes" array: {path}')
    nodes = []
    for e in j["nodes"]:
        if not isinstance(e, list) or len(e) != 2 or not all(isinstance(v, (int, float)) for v in e):
            raise RuntimeError(f"curve JSON nodes must be [x, y] pairs: {path}")
        nodes.append((float(e[0]), float(e[1])))
    return _validate(np.array(_drop_closing_duplicate(nodes), dtype=np.float64).reshape(-1, 2))


def _dump(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), allow_nan=False)


def curve_to_json(c) -> str:
    a = np.asarray(c, dtype=np.float64)
    return _dump({"nodes": [[_jnum(float(x)), _jnum(float(y))] for x, y in a], "closed": True})


def write_curve_json(path: str, c) -> None:
    try:
        with open(path, "w") as f:
            f.write(curve_to_json(c))
    except OSError as e:
        raise RuntimeError(f"cannot write file: {path}") from e


def load_curve(path: str) -> np.ndarray:  # io.cpp:107-111
    dot = path.rfind(".")
    return read_curve_json(path) if dot >= 0 and path[dot + 1:] == "json" else read_curve_csv(path)


def alignment_to_json(a) -> str:
    """a: RigidAlignment (api) or an alignment record (structured array row)."""
    get = (lambda k: getattr(a, k)) if hasattr(a, "shift") and not hasattr(a, "dtype") else (lambda k: a[k])
    return _dump({"shift": int(get("shift")), "t0": _jnum(float(get("t0"))), "theta": _jnum(float(get("theta"))),
                  "trace": _jnum(float(get("trace"))), "energy": _jnum(float(get("energy")))})


def elastic_to_json(m) -> str:
    """m: ElasticMatch (api)."""
    return _dump({"t0": _jnum(m.t0), "theta": _jnum(m.theta), "gamma": [_jnum(float(v)) for v in m.gamma],
                  "distance": _jnum(m.distance), "iterations": int(m.iterations), "converged": bool(m.converged)})


def matrix_to_csv(names, d) -> str:  # io.cpp:133-149
    d = np.asarray(d, dtype=np.float64)
    if len(names) != d.shape[0]:
        raise ValueError("matrix_to_csv: name count mismatch")
    if d.ndim != 2 or d.shape[1] != len(names):
        raise ValueError("matrix_to_csv: ragged matrix")
    rows = ["id" + "".join("," + n for n in names)]
    for n, row in zip(names, d):
        rows.append(n + "".join("," + ("nan" if math.isnan(v) else _fmt17(v)) for v in row))
    return "\n".join(rows) + "\n"
