"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle.

* ``Oracle``     -> oracle/liboracle.so, the plain-C restatement
                    (oracle/curvalign_oracle.c).
* ``Reference``  -> oracle/_ref/libcurvalign_ref.so, the reference's own sources
                    compiled in place against the FFTW/Eigen shims (oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker / CPU baseline.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libcurvalign_ref.so")

ALIGNMENT_DTYPE = [
    ("shift", "<i8"),
    ("t0", "<f8"),
    ("theta", "<f8"),
    ("trace", "<f8"),
    ("energy", "<f8"),
    ("degenerate", "<i4"),
    ("status", "<i4"),
]

FAMILIES = {"circle": 0, "superellipse": 1, "hippopede": 2, "bumps": 3, "limacon": 4, "clover": 5,
            "fourier_random": 6}


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data


class OracleError(Exception):
    pass


def _raise(rc, what):
    if rc == 1:
        raise ValueError(what)
    if rc == 2:
        raise RuntimeError(what)
    if rc != 0:
        raise OracleError(f"{what}: status {rc}")


class _Base:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = ctypes.CDLL(path)

    def _fn(self, name, argtypes):
        f = getattr(self.lib, self.prefix + name)
        f.restype = c_int
        f.argtypes = argtypes
        return f

    # ---- common surface (both libraries export these with their prefix)
    def align(self, c1, c2, fft=True):
        a, b = _f64(c1), _f64(c2)
        out = np.zeros(1, dtype=ALIGNMENT_DTYPE)
        f = self._fn("align_fft" if fft else "align_naive", [c_void_p, c_void_p, c_int64, c_void_p])
        if a.shape != b.shape:
            raise ValueError("align: node count mismatch")
        _raise(f(_p(a), _p(b), a.shape[0], _p(out)), "align")
        return out[0]

    def correlation_all_shifts(self, c1, c2, fft=True):
        a, b = _f64(c1), _f64(c2)
        n = a.shape[0]
        out = np.zeros((n, 4))
        if self.prefix == "ref_":
            f = self._fn("correlation_all_shifts", [c_void_p, c_void_p, c_int64, c_int, c_void_p])
            _raise(f(_p(a), _p(b), n, 1 if fft else 0, _p(out)), "correlation")
        else:
            f = self._fn("correlation_all_shifts_fft" if fft else "correlation_all_shifts_naive",
                         [c_void_p, c_void_p, c_int64, c_void_p])
            _raise(f(_p(a), _p(b), n, _p(out)), "correlation")
        return out

    def cross_correlation_matrix(self, c1, c2, shift):
        a, b = _f64(c1), _f64(c2)
        out = np.zeros(4)
        f = self._fn("cross_correlation_matrix", [c_void_p, c_void_p, c_int64, c_int64, c_void_p])
        if a.shape != b.shape:
            raise ValueError("align: node count mismatch")
        _raise(f(_p(a), _p(b), a.shape[0], shift, _p(out)), "cross_correlation_matrix")
        return out

    def mismatch_energy(self, c1, c2, shift, theta):
        a, b = _f64(c1), _f64(c2)
        out = np.zeros(1)
        f = self._fn("mismatch_energy", [c_void_p, c_void_p, c_int64, c_int64, c_double, c_void_p])
        _raise(f(_p(a), _p(b), a.shape[0], shift, theta, _p(out)), "mismatch_energy")
        return float(out[0])

    def preprocess(self, c, n_out, resample=True):
        a = _f64(c)
        m = n_out if resample else a.shape[0]
        out = np.zeros((m, 2))
        f = self._fn("preprocess", [c_void_p, c_int64, c_int64, c_int, c_void_p])
        _raise(f(_p(a), a.shape[0], n_out, 1 if resample else 0, _p(out)), "preprocess")
        return out

    def resample_uniform(self, c, n_out):
        a = _f64(c)
        out = np.zeros((n_out, 2))
        f = self._fn("resample_uniform", [c_void_p, c_int64, c_int64, c_void_p])
        _raise(f(_p(a), a.shape[0], n_out, _p(out)), "resample_uniform")
        return out

    def arc_length_params(self, c):
        a = _f64(c)
        s = np.zeros(a.shape[0] + 1)
        tot = np.zeros(1)
        f = self._fn("arc_length_params", [c_void_p, c_int64, c_void_p, c_void_p])
        _raise(f(_p(a), a.shape[0], _p(s), _p(tot)), "arc_length_params")
        return s, float(tot[0])

    def curve_length(self, c):
        a = _f64(c)
        out = np.zeros(1)
        f = self._fn("curve_length", [c_void_p, c_int64, c_void_p])
        _raise(f(_p(a), a.shape[0], _p(out)), "curve_length")
        return float(out[0])

    def centroid(self, c):
        a = _f64(c)
        out = np.zeros(2)
        f = self._fn("centroid", [c_void_p, c_int64, c_void_p])
        _raise(f(_p(a), a.shape[0], _p(out)), "centroid")
        return out

    def srv_transform(self, c):
        a = _f64(c)
        out = np.zeros_like(a)
        if self.prefix == "ref_":
            h = np.zeros(1)
            f = self._fn("srv_transform", [c_void_p, c_int64, c_void_p, c_void_p])
            _raise(f(_p(a), a.shape[0], _p(out), _p(h)), "srv_transform")
        else:
            f = self._fn("srv_transform", [c_void_p, c_int64, c_void_p])
            _raise(f(_p(a), a.shape[0], _p(out)), "srv_transform")
        return out

    def srv_center(self, q):
        a = _f64(q)
        out = np.zeros_like(a)
        f = self._fn("srv_center", [c_void_p, c_int64, c_void_p])
        _raise(f(_p(a), a.shape[0], _p(out)), "srv_center")
        return out

    def batch(self, points, offsets, n_out, mode=0, resample=True, threads=1, aligned=False):
        """mode 0: preprocess+align, 1: align uniform, 2: SRV align. Returns (results, aligned)."""
        pts = _f64(points)
        offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
        pairs = (offs.shape[0] - 1) // 2
        res = np.zeros(pairs, dtype=ALIGNMENT_DTYPE)
        if aligned:
            n_al = n_out if (mode == 0 and resample) else int(offs[1] - offs[0])
            al = np.zeros((pairs, n_al, 2))
        else:
            al = None
        f = self._fn("batch", [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int, c_int, c_void_p,
                               c_void_p])
        f(_p(pts), _p(offs), pairs, n_out, 1 if resample else 0, mode, threads, _p(res),
          _p(al) if al is not None else 0)
        return res, al


class _ElasticShared:
    """apply_srv_action / elastic_energy / dp_step_cost: same C signature in both libraries."""

    def apply_srv_action(self, q, t0, theta, gamma):
        a, g = _f64(q), _f64(gamma)
        out = np.zeros_like(a)
        f = self._fn("apply_srv_action", [c_void_p, c_int64, c_double, c_double, c_void_p, c_void_p])
        _raise(f(_p(a), a.shape[0], t0, theta, _p(g), _p(out)), "apply_srv_action")
        return out

    def elastic_energy(self, q1, q2, t0, theta, gamma):
        a, b, g = _f64(q1), _f64(q2), _f64(gamma)
        out = np.zeros(1)
        f = self._fn("elastic_energy", [c_void_p, c_void_p, c_int64, c_double, c_double, c_void_p, c_void_p])
        _raise(f(_p(a), _p(b), a.shape[0], t0, theta, _p(g), _p(out)), "elastic_energy")
        return float(out[0])

    def dp_step_cost(self, q1, q2, i0, j0, di, dj):
        a, b = _f64(q1), _f64(q2)
        out = np.zeros(1)
        f = self._fn("dp_step_cost", [c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_int, c_void_p])
        _raise(f(_p(a), _p(b), a.shape[0], i0, j0, di, dj, _p(out)), "dp_step_cost")
        return float(out[0])



class _OrElasticMatch(ctypes.Structure):
    _fields_ = [("t0", c_double), ("theta", c_double), ("energy", c_double), ("distance", c_double),
                ("iterations", c_int32), ("converged", c_int32), ("gamma", c_void_p)]


class Oracle(_ElasticShared, _Base):
    """The plain-C restatement (oracle/curvalign_oracle.c, oracle/elastic_oracle.c)."""

    prefix = "or_"

    def __init__(self, path=ORACLE_PATH):
        super().__init__(path)

    def dp_reparam_batch(self, q1, q2, max_slope=4, threads=1):
        a, b = _f64(q1), _f64(q2)
        pairs, n = a.shape[0], a.shape[1]
        g = np.zeros((pairs, n + 1))
        e = np.zeros(pairs)
        st = np.zeros(pairs, dtype=np.int32)
        f = self._fn("dp_reparam", [c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p])
        for p in range(pairs):
            ep = np.zeros(1)
            st[p] = f(_p(a[p]), _p(b[p]), n, max_slope, _p(g[p]), _p(ep))
            e[p] = ep[0] if st[p] == 0 else np.nan
        return g, e, st

    def elastic_approach1_batch(self, c1, c2, max_slope=4, n_max=512, threads=1, gamma=False):
        a, b = _f64(c1), _f64(c2)
        pairs, n = a.shape[0], a.shape[1]
        out = {k: np.full(pairs, np.nan) for k in ("distance", "energy", "t0", "theta")}
        out.update(iterations=np.zeros(pairs, dtype=np.int32), converged=np.zeros(pairs, dtype=np.int32),
                   status=np.zeros(pairs, dtype=np.int32))
        g = np.zeros((pairs, n + 1))
        f = self._fn("elastic_approach1", [c_void_p, c_void_p, c_int64, c_int, c_int64,
                                           ctypes.POINTER(_OrElasticMatch)])
        for p in range(pairs):
            m = _OrElasticMatch(gamma=g[p].ctypes.data)
            rc = f(_p(a[p]), _p(b[p]), n, max_slope, n_max, ctypes.byref(m))
            out["status"][p] = rc
            if rc == 0:
                for k in ("distance", "energy", "t0", "theta"):
                    out[k][p] = getattr(m, k)
                out["iterations"][p], out["converged"][p] = m.iterations, m.converged
        if gamma:
            out["gamma"] = g
        return out

    def elastic_approach2_batch(self, c1, c2, max_iters=30, energy_tol=1e-6, use_fft=True, max_slope=4,
                                threads=1, gamma=False):
        a, b = _f64(c1), _f64(c2)
        pairs, n = a.shape[0], a.shape[1]
        out = {k: np.full(pairs, np.nan) for k in ("distance", "energy", "t0", "theta")}
        out.update(iterations=np.zeros(pairs, dtype=np.int32), converged=np.zeros(pairs, dtype=np.int32),
                   status=np.zeros(pairs, dtype=np.int32))
        g = np.zeros((pairs, n + 1))
        f = self._fn("elastic_approach2", [c_void_p, c_void_p, c_int64, c_int, c_double, c_int, c_int,
                                           ctypes.POINTER(_OrElasticMatch)])
        for p in range(pairs):
            m = _OrElasticMatch(gamma=g[p].ctypes.data)
            rc = f(_p(a[p]), _p(b[p]), n, max_iters, energy_tol, 1 if use_fft else 0, max_slope, ctypes.byref(m))
            out["status"][p] = rc
            if rc == 0:
                for k in ("distance", "energy", "t0", "theta"):
                    out[k][p] = getattr(m, k)
                out["iterations"][p], out["converged"][p] = m.iterations, m.converged
        if gamma:
            out["gamma"] = g
        return out

    def spline(self, x, y, xq):
        """Second derivatives + evaluation of the periodic spline at xq."""
        x, y, xq = _f64(x), _f64(y), _f64(xq)
        m = np.zeros_like(x)
        f = self._fn("spline_second_derivs", [c_void_p, c_void_p, c_int64, c_void_p])
        _raise(f(_p(x), _p(y), x.shape[0], _p(m)), "spline")
        ev = self.lib.or_spline_eval
        ev.restype = c_double
        ev.argtypes = [c_void_p, c_void_p, c_void_p, c_int64, c_double]
        return np.array([ev(_p(x), _p(y), _p(m), x.shape[0], float(t)) for t in xq])

    def optimal_rotation(self, a4, svd=True):
        a = _f64(a4)
        th, tr = np.zeros(1), np.zeros(1)
        dg = np.zeros(1, dtype=np.int32)
        f = self._fn("optimal_rotation_svd" if svd else "optimal_rotation_closed_form",
                     [c_void_p, c_void_p, c_void_p, c_void_p])
        _raise(f(_p(a), _p(th), _p(tr), _p(dg)), "optimal_rotation")
        return float(th[0]), float(tr[0]), bool(dg[0])

    def real_dft(self, x):
        x = _f64(x)
        out = np.zeros((x.shape[0] // 2 + 1, 2))
        f = self._fn("real_dft", [c_void_p, c_int64, c_void_p])
        _raise(f(_p(x), x.shape[0], _p(out)), "real_dft")
        return out[:, 0] + 1j * out[:, 1]

    def circular_cross_correlation(self, a, b):
        a, b = _f64(a), _f64(b)
        out = np.zeros(a.shape[0])
        f = self._fn("circular_cross_correlation", [c_void_p, c_void_p, c_int64, c_void_p])
        _raise(f(_p(a), _p(b), a.shape[0], _p(out)), "circular_cross_correlation")
        return out


class Reference(_ElasticShared, _Base):
    """The reference's own code compiled in place (oracle/_ref)."""

    prefix = "ref_"

    def __init__(self, path=REF_PATH):
        super().__init__(path)

    def spline(self, x, y, xq, derivative=False):
        x, y, xq = _f64(x), _f64(y), _f64(xq)
        out = np.zeros_like(xq)
        f = self._fn("spline_eval", [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int, c_void_p])
        _raise(f(_p(x), _p(y), x.shape[0], _p(xq), xq.shape[0], 1 if derivative else 0, _p(out)), "spline")
        return out

    def optimal_rotation(self, a4, svd=True):
        a = _f64(a4)
        th, tr = np.zeros(1), np.zeros(1)
        dg = np.zeros(1, dtype=np.int32)
        f = self._fn("optimal_rotation", [c_void_p, c_int, c_void_p, c_void_p, c_void_p])
        _raise(f(_p(a), 1 if svd else 0, _p(th), _p(tr), _p(dg)), "optimal_rotation")
        return float(th[0]), float(tr[0]), bool(dg[0])

    def gen_curve(self, family, n, seed=1, harmonics=12):
        out = np.zeros((n, 2))
        f = self._fn("gen_curve", [c_int, c_int64, c_uint64, c_int, c_void_p])
        _raise(f(FAMILIES[family], n, seed, harmonics, _p(out)), "gen_curve")
        return out

    def transform_curve(self, c, start_shift, theta, warp=0, u=0.0):
        a = _f64(c)
        out = np.zeros_like(a)
        f = self._fn("transform_curve", [c_void_p, c_int64, c_double, c_double, c_int, c_double, c_void_p])
        _raise(f(_p(a), a.shape[0], start_shift, theta, warp, u, _p(out)), "transform_curve")
        return out

    def real_dft(self, x):
        x = _f64(x)
        out = np.zeros((x.shape[0] // 2 + 1, 2))
        f = self._fn("real_dft", [c_void_p, c_int64, c_void_p])
        _raise(f(_p(x), x.shape[0], _p(out)), "real_dft")
        return out[:, 0] + 1j * out[:, 1]

    def circular_cross_correlation(self, a, b):
        a, b = _f64(a), _f64(b)
        out = np.zeros(a.shape[0])
        f = self._fn("circular_cross_correlation", [c_void_p, c_int64, c_void_p, c_int64, c_void_p])
        _raise(f(_p(a), a.shape[0], _p(b), b.shape[0], _p(out)), "circular_cross_correlation")
        return out

    def allpairs(self, curves, row_begin, row_end, threads=1):
        c = _f64(curves)
        m, n = c.shape[0], c.shape[1]
        rows = row_end - row_begin
        e = np.zeros((rows, m))
        k = np.zeros((rows, m), dtype=np.int64)
        th = np.zeros((rows, m))
        f = self._fn("allpairs", [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p,
                                  c_void_p])
        _raise(f(_p(c), m, n, row_begin, row_end, threads, _p(e), _p(k), _p(th)), "allpairs")
        return e, k, th


    def dp_reparam_batch(self, q1, q2, max_slope=4, threads=1):
        a, b = _f64(q1), _f64(q2)
        pairs, n = a.shape[0], a.shape[1]
        g = np.zeros((pairs, n + 1))
        e = np.zeros(pairs)
        st = np.zeros(pairs, dtype=np.int32)
        f = self._fn("dp_reparam_batch", [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int, c_void_p, c_void_p,
                                          c_void_p])
        f(_p(a), _p(b), pairs, n, max_slope, threads, _p(g), _p(e), _p(st))
        return g, e, st

    def elastic_approach2_batch(self, c1, c2, max_iters=30, energy_tol=1e-6, use_fft=True, max_slope=4,
                                threads=1, gamma=False):
        a, b = _f64(c1), _f64(c2)
        pairs, n = a.shape[0], a.shape[1]
        out = {k: np.zeros(pairs) for k in ("distance", "energy", "t0", "theta")}
        g = np.zeros((pairs, n + 1)) if gamma else None
        it = np.zeros(pairs, dtype=np.int32)
        cv = np.zeros(pairs, dtype=np.int32)
        st = np.zeros(pairs, dtype=np.int32)
        tr = np.zeros((pairs, max_iters + 1))
        f = self._fn("elastic_approach2_batch", [c_void_p, c_void_p, c_int64, c_int64, c_int, c_double, c_int, c_int,
                                                 c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                                 c_void_p, c_void_p, c_void_p])
        f(_p(a), _p(b), pairs, n, max_iters, energy_tol, 1 if use_fft else 0, max_slope, threads,
          _p(out["distance"]), _p(out["energy"]), _p(out["t0"]), _p(out["theta"]), _p(g) if gamma else None,
          _p(it), _p(cv), _p(st), _p(tr))
        out.update(iterations=it, converged=cv, status=st, energy_trace=tr)
        if gamma:
            out["gamma"] = g
        return out

    def distance_matrix(self, curves, n, method=2, max_iters=30, energy_tol=1e-6, max_slope=4, threads=1):
        c = _f64(curves)
        k, n_in = c.shape[0], c.shape[1]
        out = np.zeros((k, k))
        f = self._fn("distance_matrix", [c_void_p, c_int64, c_int64, c_int64, c_int, c_int, c_double, c_int,
                                         c_int, c_void_p])
        _raise(f(_p(c), k, n_in, n, method, max_iters, energy_tol, max_slope, threads, _p(out)), "distance_matrix")
        return out

    def distance_matrix_approach2(self, curves, n, max_iters=30, energy_tol=1e-6, max_slope=4, threads=1):
        return self.distance_matrix(curves, n, 2, max_iters, energy_tol, max_slope, threads)

    def elastic_approach1_batch(self, c1, c2, max_slope=4, n_max=512, threads=1, gamma=False):
        a, b = _f64(c1), _f64(c2)
        pairs, n = a.shape[0], a.shape[1]
        out = {k: np.zeros(pairs) for k in ("distance", "energy", "t0", "theta")}
        g = np.zeros((pairs, n + 1)) if gamma else None
        it, cv, st = (np.zeros(pairs, dtype=np.int32) for _ in range(3))
        f = self._fn("elastic_approach1_batch", [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int64, c_int,
                                                 c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                                 c_void_p, c_void_p])
        f(_p(a), _p(b), pairs, n, max_slope, n_max, threads, _p(out["distance"]), _p(out["energy"]), _p(out["t0"]),
          _p(out["theta"]), _p(g) if gamma else None, _p(it), _p(cv), _p(st))
        out.update(iterations=it, converged=cv, status=st)
        if gamma:
            out["gamma"] = g
        return out


class _RefFormats:
    """proj/src/io.cpp through oracle/_ref (strings returned via a buffer)."""

    def _str(self, name, argtypes, *args):
        buf = ctypes.create_string_buffer(1 << 22)
        ln = np.zeros(1, dtype=np.int64)
        f = self._fn(name, argtypes + [c_void_p, c_int64, c_void_p])
        _raise(f(*args, ctypes.addressof(buf), len(buf), _p(ln)), name)
        return buf.raw[: int(ln[0])].decode()

    def load_curve(self, path):
        out = np.zeros((1 << 20, 2))
        n = np.zeros(1, dtype=np.int64)
        f = self._fn("load_curve", [ctypes.c_char_p, c_void_p, c_int64, c_void_p])
        _raise(f(path.encode(), _p(out), out.shape[0], _p(n)), "load_curve")
        return out[: int(n[0])].copy()

    def write_curve(self, path, c, json=False):
        a = _f64(c)
        f = self._fn("write_curve", [ctypes.c_char_p, c_void_p, c_int64, c_int])
        _raise(f(path.encode(), _p(a), a.shape[0], 1 if json else 0), "write_curve")

    def curve_to_csv(self, c):
        a = _f64(c)
        return self._str("curve_to_csv", [c_void_p, c_int64], _p(a), a.shape[0])

    def curve_to_json(self, c):
        a = _f64(c)
        return self._str("curve_to_json", [c_void_p, c_int64], _p(a), a.shape[0])

    def alignment_to_json(self, rec):
        r = np.ascontiguousarray(np.asarray(rec, dtype=ALIGNMENT_DTYPE).reshape(1))
        return self._str("alignment_to_json", [c_void_p], r.ctypes.data)

    def elastic_to_json(self, t0, theta, gamma, distance, iterations, converged):
        g = _f64(gamma)
        return self._str("elastic_to_json", [c_double, c_double, c_void_p, c_int64, c_double, c_int, c_int],
                         t0, theta, _p(g), g.shape[0], distance, int(iterations), int(converged))

    def matrix_to_csv(self, names, d):
        m = _f64(d)
        return self._str("matrix_to_csv", [ctypes.c_char_p, c_int64, c_void_p], "\n".join(names).encode(),
                         m.shape[0], _p(m))


Reference.__bases__ = (_RefFormats,) + Reference.__bases__


def reference_available() -> bool:
    return os.path.exists(REF_PATH)
