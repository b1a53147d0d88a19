"""CPU: curve / result file formats (paper_2501_17779_b200.formats) against the
reference's own io.cpp compiled in place (oracle/_ref): byte-identical writers,
readers that accept exactly what the reference accepts. Cases restate
proj/tests/test_io_cli.cpp:50-135 (the CLI cases there are out of scope)."""
import json
import os

import numpy as np
import pytest

from paper_2501_17779_b200 import formats as F
from paper_2501_17779_b200.api import ElasticMatch

FAM = ["circle", "superellipse", "hippopede", "bumps", "limacon", "clover", "fourier_random"]


@pytest.fixture
def tmp(tmp_path):
    return lambda name: str(tmp_path / name)


def _write(path, text):
    with open(path, "w") as f:
        f.write(text)


@pytest.mark.parametrize("fam", FAM)
def test_writers_byte_identical(reference, fam):
    c = reference.gen_curve(fam, 37)
    assert F.curve_to_csv(c) == reference.curve_to_csv(c)
    assert F.curve_to_json(c) == reference.curve_to_json(c)


def test_writers_special_values(reference):
    c = np.array([[0.1, -0.0], [1e-7, 1e20], [123456.0, -2.5e-300], [3.0, 1.0 / 3.0]])
    assert F.curve_to_csv(c) == reference.curve_to_csv(c)
    assert json.loads(F.curve_to_json(c)) == json.loads(reference.curve_to_json(c))


def test_round_trips_both_ways(reference, tmp):  # test_io_cli.cpp:50-72
    c = reference.gen_curve("limacon", 32)
    for ext, json_ in (("csv", False), ("json", True)):
        p1, p2 = tmp(f"ours.{ext}"), tmp(f"ref.{ext}")
        (F.write_curve_json if json_ else F.write_curve_csv)(p1, c)
        reference.write_curve(p2, c, json=json_)
        np.testing.assert_array_equal(reference.load_curve(p1), c)  # ours -> reference reader
        np.testing.assert_array_equal(F.load_curve(p2), c)  # reference -> our reader
        np.testing.assert_array_equal(F.load_curve(p1), c)


def test_csv_header_and_closing_duplicate(reference, tmp):  # test_io_cli.cpp:74-82
    p = tmp("headered.csv")
    _write(p, "x,y\n1,0\n0,1\n-1,0\n0,-1\n1,0\n")
    c = F.read_curve_csv(p)
    assert c.shape == (4, 2) and c[0, 0] == 1.0 and c[3, 1] == -1.0
    np.testing.assert_array_equal(c, reference.load_curve(p))


@pytest.mark.parametrize("text", ["1,2\nthree\n4,5\n6,7\n", "x,y\n1,2\nalpha,beta\n3,4\n5,6\n", "1,2\n3,4\n",
                                  "1,2\n3,\n4,5\n6,7\n", "1,2\n3,4\n5,6\nnan,1\n"])
def test_csv_rejects_like_reference(reference, tmp, text):  # test_io_cli.cpp:84-98
    p = tmp("bad.csv")
    _write(p, text)
    with pytest.raises(Exception):
        reference.load_curve(p)
    with pytest.raises((RuntimeError, ValueError)):
        F.read_curve_csv(p)


def test_csv_lenient_cells_like_reference(reference, tmp):
    """std::stod semantics: blanks, trailing junk and extra columns accepted."""
    p = tmp("lenient.csv")
    _write(p, " 1,0 \n0 ,1x\n-1,0,9\n0,-1\r\n\n\r\n")
    np.testing.assert_array_equal(F.read_curve_csv(p), reference.load_curve(p))


def test_missing_file(tmp):
    with pytest.raises(RuntimeError):
        F.read_curve_csv(tmp("does_not_exist.csv"))


@pytest.mark.parametrize("text", ['{"points": [[0, 0]]}', '{"nodes": [[0, 0, 0], [1, 1]]}', "[1, 2]",
                                  '{"nodes": [[0, 0], [1, "a"], [2, 2], [3, 3]]}'])
def test_json_schema_like_reference(reference, tmp, text):  # test_io_cli.cpp:100-108
    p = tmp("bad.json")
    _write(p, text)
    with pytest.raises(Exception):
        reference.load_curve(p)
    with pytest.raises((RuntimeError, ValueError)):
        F.read_curve_json(p)


def test_load_curve_dispatch(reference, tmp):  # test_io_cli.cpp:110-118
    c = reference.gen_curve("bumps", 20)
    F.write_curve_json(tmp("d.json"), c)
    F.write_curve_csv(tmp("d.csv"), c)
    assert F.load_curve(tmp("d.json")).shape == (20, 2) and F.load_curve(tmp("d.csv")).shape == (20, 2)


def test_result_json_and_matrix_csv(reference):  # test_io_cli.cpp:120-135
    from pyoracle import ALIGNMENT_DTYPE

    rec = np.zeros(1, dtype=ALIGNMENT_DTYPE)[0]
    rec["shift"], rec["t0"], rec["theta"], rec["trace"], rec["energy"] = 29, 29 / 96, -1.2345678901234567, 21.5, 3e-9
    assert F.alignment_to_json(rec) == reference.alignment_to_json(rec)
    g = np.sort(np.random.default_rng(0).uniform(0, 1, 9))
    g[0], g[-1] = 0.0, 1.0
    m = ElasticMatch(t0=0.25, theta=0.5, gamma=g, energy=0.04, distance=0.2, iterations=3, converged=True)
    assert F.elastic_to_json(m) == reference.elastic_to_json(0.25, 0.5, g, 0.2, 3, 1)
    names = ["a", "b"]
    d = [[0.0, 0.5], [np.nan, 0.0]]
    assert F.matrix_to_csv(names, d) == reference.matrix_to_csv(names, d) == "id,a,b\na,0,0.5\nb,nan,0\n"
    with pytest.raises(ValueError):
        F.matrix_to_csv(["a"], d)
    rng = np.random.default_rng(1)
    big = rng.standard_normal((5, 5))
    nm = [f"c{i}" for i in range(5)]
    assert F.matrix_to_csv(nm, big) == reference.matrix_to_csv(nm, big)
