"""Python host mirror of the reference's alignment API over the C ABI.

Names and argument meaning follow /root/reference/proj/include/curvalign/:
``align_fft`` (rigid_align.hpp:44-51), ``preprocess`` (curve.hpp:47-48),
``srv_transform``/``srv_center`` pattern (srv.hpp:23-27). Errors map to the
exception classes the reference throws (std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError, std::bad_alloc -> MemoryError).

Two calling conventions:

* numpy arrays (host memory): the synchronous ``*_host`` C entry points copy
  to the GPU, run the kernels and copy back;
* torch CUDA tensors (device memory): the asynchronous device entry points run
  on torch's current stream; results stay on the device.

Curves are ``(n, 2)`` float64 arrays (x, y) — the byte layout of
``curvalign::Point2`` — and batches are ``(pairs, n, 2)``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import ALIGNMENT_DTYPE, check

try:  # torch is plumbing only (device memory + streams)
    import torch
except Exception:  # pragma: no cover
    torch = None


@dataclass
class RigidAlignment:
    """Mirror of curvalign::RigidAlignment (rigid_align.hpp:16-23)."""

    shift: int
    t0: float
    theta: float
    trace: float
    energy: float
    degenerate: bool


def _is_cuda_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _f64c(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a is not None and a.size else (a.ctypes.data if a is not None else 0)


def _tptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def _stream_of(t) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def decode_results(raw) -> np.ndarray:
    """Alignment results (device tensor of bytes or numpy buffer) -> structured array."""
    if _is_cuda_tensor(raw):
        raw = raw.cpu().numpy()
    return np.frombuffer(np.ascontiguousarray(raw).tobytes(), dtype=ALIGNMENT_DTYPE)


def _result_from_record(r) -> RigidAlignment:
    return RigidAlignment(
        shift=int(r["shift"]),
        t0=float(r["t0"]),
        theta=float(r["theta"]),
        trace=float(r["trace"]),
        energy=float(r["energy"]),
        degenerate=bool(r["degenerate"]),
    )


def _raise_pair_status(res: np.ndarray) -> None:
    bad = np.nonzero(res["status"] != 0)[0]
    if bad.size:
        st = int(res["status"][bad[0]])
        msg = f"pair {int(bad[0])}: status {st}"
        if st == _native.CVA_INVALID_ARGUMENT:
            raise ValueError(msg)
        if st == _native.CVA_RUNTIME_ERROR:
            raise RuntimeError(msg)
        raise _native.CurvalignError(msg)


# --------------------------------------------------------------- align_fft


def align_fft_batch(c1, c2, return_aligned: bool = False):
    """align_fft over a batch of pre-sampled pairs (rigid_align.cpp:204-208).

    c1, c2: ``(pairs, n, 2)`` float64, numpy (host) or CUDA tensor (device).
    Returns ``(results, aligned)``: a structured array (host) or a ``(pairs, 48)``
    uint8 device tensor (decode with :func:`decode_results`), and the aligned
    curves ``R c2[(l + shift) mod n]`` or None.
    """
    lib = _native.load()
    if _is_cuda_tensor(c1):
        if c1.shape != c2.shape or c1.dim() != 3 or c1.shape[2] != 2:
            raise ValueError("align: node count mismatch")
        c1 = c1.contiguous().to(torch.float64)
        c2 = c2.contiguous().to(torch.float64)
        pairs, n = c1.shape[0], c1.shape[1]
        out = torch.empty((pairs, 48), dtype=torch.uint8, device=c1.device)
        al = torch.empty_like(c2) if return_aligned else None
        check(lib.cva_align_batch(c1.data_ptr(), c2.data_ptr(), pairs, n, out.data_ptr(),
                                  _tptr(al), _stream_of(c1)))
        return out, al
    a, b = _f64c(c1), _f64c(c2)
    if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 2:
        raise ValueError("align: node count mismatch")
    pairs, n = a.shape[0], a.shape[1]
    res = np.zeros(pairs, dtype=ALIGNMENT_DTYPE)
    al = np.empty_like(b) if return_aligned else None
    check(lib.cva_align_batch_host(_ptr(a), _ptr(b), pairs, n, res.ctypes.data,
                                   al.ctypes.data if al is not None else 0))
    return res, al


def align_fft(c1, c2) -> RigidAlignment:
    """Single-pair drop-in for curvalign::align_fft (rigid_align.hpp:45,50)."""
    a, b = _f64c(c1), _f64c(c2)
    if a.ndim != 2 or b.ndim != 2 or a.shape[0] != b.shape[0]:
        raise ValueError("align: node count mismatch")
    res, _ = align_fft_batch(a[None], b[None])
    _raise_pair_status(res)
    return _result_from_record(res[0])


def aligned_curve(c1, c2):
    """align_fft plus the aligned second curve R c2[(l + shift) mod N]."""
    a, b = _f64c(c1), _f64c(c2)
    if a.ndim != 2 or b.ndim != 2 or a.shape[0] != b.shape[0]:
        raise ValueError("align: node count mismatch")
    res, al = align_fft_batch(a[None], b[None], return_aligned=True)
    _raise_pair_status(res)
    return _result_from_record(res[0]), al[0]


# -------------------------------------------------------------- preprocess


def ragged(curves) -> tuple[np.ndarray, np.ndarray]:
    """List of (n_i, 2) arrays -> (points (sum n_i, 2), offsets (len+1,) int64)."""
    offs = np.zeros(len(curves) + 1, dtype=np.int64)
    for i, c in enumerate(curves):
        offs[i + 1] = offs[i] + np.asarray(c).shape[0]
    pts = np.concatenate([_f64c(c).reshape(-1, 2) for c in curves]) if curves else np.zeros((0, 2))
    return np.ascontiguousarray(pts), offs


def preprocess_batch(points, offsets, n_out: int, resample: bool = True, max_n_in: int = 0):
    """preprocess (curve.cpp:93-97) of a ragged batch: returns (curves, status).

    numpy inputs: curves is ``(count, n_out, 2)`` (resample) or the input's
    ragged ``(total, 2)`` layout (no resample). CUDA tensors: same on device.
    """
    lib = _native.load()
    if _is_cuda_tensor(points):
        count = offsets.shape[0] - 1
        total = points.shape[0]
        out = torch.empty((count, n_out, 2) if resample else (total, 2), dtype=torch.float64,
                          device=points.device)
        st = torch.empty(count, dtype=torch.int32, device=points.device)
        check(lib.cva_preprocess_batch(points.data_ptr(), offsets.data_ptr(), count, int(max_n_in),
                                       int(n_out), 1 if resample else 0, out.data_ptr(),
                                       st.data_ptr(), _stream_of(points)))
        return out, st
    pts = _f64c(points)
    offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    count = offs.shape[0] - 1
    out = np.empty((count, n_out, 2) if resample else pts.shape, dtype=np.float64)
    st = np.zeros(count, dtype=np.int32)
    check(lib.cva_preprocess_batch_host(_ptr(pts), offs.ctypes.data, count, int(n_out),
                                        1 if resample else 0, out.ctypes.data, st.ctypes.data))
    return out, st


def preprocess(curve, n_out: int, resample: bool = True) -> np.ndarray:
    """Drop-in for curvalign::preprocess (curve.hpp:47-48): (n, 2) -> (n_out or n, 2)."""
    c = _f64c(curve)
    if c.ndim != 2 or c.shape[1] != 2:
        raise ValueError("curve: expected (n, 2) nodes")
    if resample and n_out < 8:
        raise ValueError("resample: need at least 8 output nodes")
    pts, offs = ragged([c])
    out, st = preprocess_batch(pts, offs, n_out, resample)
    if st[0] == _native.CVA_INVALID_ARGUMENT:
        raise ValueError("curve: invalid input (too few / non-finite / coincident nodes)")
    if st[0] != 0:
        raise RuntimeError(f"preprocess: status {int(st[0])}")
    return out[0] if resample else out


def resample_batch(points, offsets, n_out: int, max_n_in: int = 0):
    """resample_uniform (curve.cpp:67-91) of a ragged batch: returns (curves, status)."""
    lib = _native.load()
    if _is_cuda_tensor(points):
        count = offsets.shape[0] - 1
        out = torch.empty((count, n_out, 2), dtype=torch.float64, device=points.device)
        st = torch.empty(count, dtype=torch.int32, device=points.device)
        check(lib.cva_resample_batch(points.data_ptr(), offsets.data_ptr(), count, int(max_n_in),
                                     int(n_out), out.data_ptr(), st.data_ptr(), _stream_of(points)))
        return out, st
    pts = _f64c(points)
    offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    count = offs.shape[0] - 1
    out = np.empty((count, n_out, 2), dtype=np.float64)
    st = np.zeros(count, dtype=np.int32)
    check(lib.cva_resample_batch_host(_ptr(pts), offs.ctypes.data, count, int(n_out),
                                      out.ctypes.data, st.ctypes.data))
    return out, st


def resample_uniform(curve, n_out: int) -> np.ndarray:
    """Drop-in for curvalign::resample_uniform (curve.hpp:44-45)."""
    c = _f64c(curve)
    if c.ndim != 2 or c.shape[1] != 2:
        raise ValueError("curve: expected (n, 2) nodes")
    if n_out < 8:
        raise ValueError("resample: need at least 8 output nodes")
    pts, offs = ragged([c])
    out, st = resample_batch(pts, offs, n_out)
    if st[0] == _native.CVA_INVALID_ARGUMENT:
        raise ValueError("curve: invalid input (too few / non-finite / coincident nodes)")
    if st[0] != 0:
        raise RuntimeError(f"resample: status {int(st[0])}")
    return out[0]


def preprocess_align_batch(points, offsets, n_out: int, max_n_in: int = 0,
                           return_aligned: bool = False):
    """Fused C1 path: pair p = (curve 2p, curve 2p+1): preprocess both to n_out
    nodes and align. Returns (results, aligned) like :func:`align_fft_batch`."""
    lib = _native.load()
    if _is_cuda_tensor(points):
        pairs = (offsets.shape[0] - 1) // 2
        out = torch.empty((pairs, 48), dtype=torch.uint8, device=points.device)
        al = (torch.empty((pairs, n_out, 2), dtype=torch.float64, device=points.device)
              if return_aligned else None)
        check(lib.cva_preprocess_align_batch(points.data_ptr(), offsets.data_ptr(), pairs,
                                             int(max_n_in), int(n_out), 1, out.data_ptr(),
                                             _tptr(al), _stream_of(points)))
        return out, al
    pts = _f64c(points)
    offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    pairs = (offs.shape[0] - 1) // 2
    res = np.zeros(pairs, dtype=ALIGNMENT_DTYPE)
    al = np.empty((pairs, n_out, 2)) if return_aligned else None
    check(lib.cva_preprocess_align_batch_host(_ptr(pts), offs.ctypes.data, pairs, int(n_out), 1,
                                              res.ctypes.data,
                                              al.ctypes.data if al is not None else 0))
    return res, al


def srv_align_batch(c1, c2, return_aligned: bool = False):
    """SRV-space alignment: align_fft(srv_center(srv_transform(c1)).q,
    srv_center(srv_transform(c2)).q) per pair (srv.cpp:71-98, elastic.cpp:138-139)."""
    lib = _native.load()
    if _is_cuda_tensor(c1):
        c1 = c1.contiguous()
        c2 = c2.contiguous()
        pairs, n = c1.shape[0], c1.shape[1]
        out = torch.empty((pairs, 48), dtype=torch.uint8, device=c1.device)
        al = torch.empty_like(c2) if return_aligned else None
        check(lib.cva_srv_align_batch(c1.data_ptr(), c2.data_ptr(), pairs, n, out.data_ptr(),
                                      _tptr(al), _stream_of(c1)))
        return out, al
    a, b = _f64c(c1), _f64c(c2)
    if a.shape != b.shape or a.ndim != 3:
        raise ValueError("srv: size mismatch")
    pairs, n = a.shape[0], a.shape[1]
    res = np.zeros(pairs, dtype=ALIGNMENT_DTYPE)
    al = np.empty_like(b) if return_aligned else None
    check(lib.cva_srv_align_batch_host(_ptr(a), _ptr(b), pairs, n, res.ctypes.data,
                                       al.ctypes.data if al is not None else 0))
    return res, al


# --------------------------------------------------------------- all pairs


def allpairs(curves, row_begin: int = 0, row_end: int | None = None):
    """All ordered pairs of pre-sampled curves (BASELINE config C2).

    curves: ``(count, n, 2)`` float64 (preprocessed). Returns
    ``(energy, shift, theta)`` matrices of rows [row_begin, row_end) x count,
    cell (r, j) = align_fft(curves[row_begin + r], curves[j]). numpy in ->
    numpy out (synchronous); CUDA tensor in -> CUDA tensors out (stream-ordered).
    """
    lib = _native.load()
    if _is_cuda_tensor(curves):
        c = curves.contiguous()
        count, n = c.shape[0], c.shape[1]
        re = count if row_end is None else row_end
        rows = re - row_begin
        e = torch.empty((rows, count), dtype=torch.float64, device=c.device)
        k = torch.empty((rows, count), dtype=torch.int32, device=c.device)
        th = torch.empty((rows, count), dtype=torch.float64, device=c.device)
        check(lib.cva_allpairs(c.data_ptr(), count, n, row_begin, re, e.data_ptr(), k.data_ptr(),
                               th.data_ptr(), _stream_of(c)))
        return e, k, th
    c = _f64c(curves)
    count, n = c.shape[0], c.shape[1]
    re = count if row_end is None else row_end
    rows = re - row_begin
    e = np.empty((rows, count))
    k = np.empty((rows, count), dtype=np.int32)
    th = np.empty((rows, count))
    check(lib.cva_allpairs_host(_ptr(c), count, n, row_begin, re, e.ctypes.data, k.ctypes.data,
                                th.ctypes.data))
    return e, k, th


def preprocess_align_uniform(c1, c2, return_aligned: bool = False):
    """preprocess(resample=false) of both curves + align_fft for equal-size
    pairs (BASELINE C0 / C3). Same conventions as :func:`align_fft_batch`."""
    lib = _native.load()
    if _is_cuda_tensor(c1):
        c1 = c1.contiguous()
        c2 = c2.contiguous()
        pairs, n = c1.shape[0], c1.shape[1]
        out = torch.empty((pairs, 48), dtype=torch.uint8, device=c1.device)
        al = torch.empty_like(c2) if return_aligned else None
        check(lib.cva_preprocess_align_uniform(c1.data_ptr(), c2.data_ptr(), pairs, n, out.data_ptr(),
                                               _tptr(al), _stream_of(c1)))
        return out, al
    a, b = _f64c(c1), _f64c(c2)
    if a.shape != b.shape or a.ndim != 3:
        raise ValueError("align: node count mismatch")
    pairs, n = a.shape[0], a.shape[1]
    res = np.zeros(pairs, dtype=ALIGNMENT_DTYPE)
    al = np.empty_like(b) if return_aligned else None
    check(lib.cva_preprocess_align_uniform_host(_ptr(a), _ptr(b), pairs, n, res.ctypes.data,
                                                al.ctypes.data if al is not None else 0))
    return res, al


# --------------------------------------------------------------- elastic (SRV) matching


@dataclass
class ElasticMatch:
    """Mirror of ``curvalign::ElasticMatch`` (proj/include/curvalign/elastic.hpp:23-32)
    without the energy trace."""

    t0: float
    theta: float
    gamma: np.ndarray
    energy: float
    distance: float
    iterations: int
    converged: bool


def dp_reparam_batch(q1, q2, max_slope: int = 4):
    """dp_reparam (srv.cpp:180-257) per pair of SRV sample arrays ``(pairs, n, 2)``.

    Returns ``(gamma (pairs, n+1), energy (pairs,), status (pairs,))``; numpy in ->
    numpy out, CUDA tensors in -> CUDA tensors out. Bitwise the reference's DP."""
    lib = _native.load()
    if _is_cuda_tensor(q1):
        a, b = q1.contiguous(), q2.contiguous()
        pairs, n = a.shape[0], a.shape[1]
        g = torch.empty((pairs, n + 1), dtype=torch.float64, device=a.device)
        e = torch.empty(pairs, dtype=torch.float64, device=a.device)
        st = torch.empty(pairs, dtype=torch.int32, device=a.device)
        check(lib.cva_dp_reparam_batch(a.data_ptr(), b.data_ptr(), pairs, n, max_slope, g.data_ptr(),
                                       e.data_ptr(), st.data_ptr(), _stream_of(a)))
        return g, e, st
    a, b = _f64c(q1), _f64c(q2)
    if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 2:
        raise ValueError("dp: size mismatch")
    pairs, n = a.shape[0], a.shape[1]
    g = np.empty((pairs, n + 1))
    e = np.empty(pairs)
    st = np.empty(pairs, dtype=np.int32)
    check(lib.cva_dp_reparam_batch_host(_ptr(a), _ptr(b), pairs, n, max_slope, g.ctypes.data, e.ctypes.data,
                                        st.ctypes.data))
    return g, e, st


def dp_reparam(q1, q2, max_slope: int = 4):
    """Single-pair dp_reparam: returns ``(gamma, energy)``; RuntimeError if no
    admissible path (srv.cpp:233)."""
    g, e, st = dp_reparam_batch(np.asarray(q1)[None], np.asarray(q2)[None], max_slope)
    if st[0] != 0:
        raise RuntimeError("dp: no admissible path")
    return g[0], float(e[0])


def _elastic_batch(approach, c1, c2, max_iters, energy_tol, max_slope, n_max_approach1, return_gamma,
                   use_fft=True):
    lib = _native.load()
    if _is_cuda_tensor(c1):
        a, b = c1.contiguous(), c2.contiguous()
        pairs, n = a.shape[0], a.shape[1]
        dev = a.device
        out = {k: torch.empty(pairs, dtype=torch.float64, device=dev) for k in ("distance", "energy", "t0", "theta")}
        for k in ("iterations", "converged", "status"):
            out[k] = torch.empty(pairs, dtype=torch.int32, device=dev)
        g = torch.empty((pairs, n + 1), dtype=torch.float64, device=dev) if return_gamma else None
        ptrs = [out[k].data_ptr() for k in ("distance", "energy", "t0", "theta")] + [_tptr(g)] + \
            [out[k].data_ptr() for k in ("iterations", "converged", "status")]
        if approach == 1:
            check(lib.cva_elastic_approach1_batch(a.data_ptr(), b.data_ptr(), pairs, n, max_slope, n_max_approach1,
                                                  *ptrs, _stream_of(a)))
        else:
            tr = torch.empty((pairs, max_iters + 1), dtype=torch.float64, device=dev)
            check(lib.cva_elastic_approach2_batch_ex(a.data_ptr(), b.data_ptr(), pairs, n, max_iters, energy_tol,
                                                     max_slope, int(bool(use_fft)), *ptrs, tr.data_ptr(),
                                                     _stream_of(a)))
            out["energy_trace"] = tr
    else:
        a, b = _f64c(c1), _f64c(c2)
        if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 2:
            raise ValueError("elastic: node count mismatch")
        pairs, n = a.shape[0], a.shape[1]
        out = {k: np.empty(pairs) for k in ("distance", "energy", "t0", "theta")}
        for k in ("iterations", "converged", "status"):
            out[k] = np.empty(pairs, dtype=np.int32)
        g = np.empty((pairs, n + 1)) if return_gamma else None
        ptrs = [out[k].ctypes.data for k in ("distance", "energy", "t0", "theta")] + \
            [g.ctypes.data if g is not None else 0] + [out[k].ctypes.data for k in ("iterations", "converged", "status")]
        if approach == 1:
            check(lib.cva_elastic_approach1_batch_host(_ptr(a), _ptr(b), pairs, n, max_slope, n_max_approach1, *ptrs))
        else:
            tr = np.empty((pairs, max_iters + 1))
            check(lib.cva_elastic_approach2_batch_ex_host(_ptr(a), _ptr(b), pairs, n, max_iters, energy_tol,
                                                          max_slope, int(bool(use_fft)), *ptrs, tr.ctypes.data))
            out["energy_trace"] = tr
    if return_gamma:
        out["gamma"] = g
    return out


def elastic_approach2_batch(c1, c2, max_iters: int = 30, energy_tol: float = 1e-6, max_slope: int = 4,
                            return_gamma: bool = False, use_fft: bool = True):
    """elastic_distance_approach2 (elastic.cpp:102-174) per pair of preprocessed
    curves ``(pairs, n, 2)``. Returns a dict of per-pair arrays: distance,
    energy, t0, theta, iterations, converged, status, energy_trace (pairs x
    (max_iters+1), NaN-padded) (+ gamma). numpy in -> numpy out; CUDA tensors in ->
    CUDA tensors out (stream-ordered). use_fft (ElasticOptions::use_fft): the
    rigid steps by the FFT correlation (align_fft) or the direct sums (align_naive)."""
    return _elastic_batch(2, c1, c2, max_iters, energy_tol, max_slope, 512, return_gamma, use_fft)


def elastic_approach1_batch(c1, c2, max_slope: int = 4, n_max_approach1: int = 512, return_gamma: bool = False):
    """elastic_distance_approach1 (elastic.cpp:62-100): exhaustive over start
    shifts, one DP each. Same outputs as :func:`elastic_approach2_batch`."""
    return _elastic_batch(1, c1, c2, 0, 0.0, max_slope, n_max_approach1, return_gamma)


def _match(r):
    st = int(r["status"][0])
    if st == _native.CVA_INVALID_ARGUMENT:
        raise ValueError("elastic: invalid input")
    if st == _native.CVA_RUNTIME_ERROR:
        raise RuntimeError("dp: no admissible path")
    return ElasticMatch(t0=float(r["t0"][0]), theta=float(r["theta"][0]), gamma=r["gamma"][0],
                        energy=float(r["energy"][0]), distance=float(r["distance"][0]),
                        iterations=int(r["iterations"][0]), converged=bool(r["converged"][0]))


def elastic_distance_approach2(c1, c2, max_iters: int = 30, energy_tol: float = 1e-6,
                               max_slope: int = 4, use_fft: bool = True) -> ElasticMatch:
    """Single pair (reference name and exceptions: ValueError for invalid input,
    RuntimeError for a DP without admissible path)."""
    a, b = np.asarray(c1, dtype=np.float64), np.asarray(c2, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("elastic: node count mismatch")
    return _match(elastic_approach2_batch(a[None], b[None], max_iters, energy_tol, max_slope, return_gamma=True,
                                          use_fft=use_fft))


def elastic_distance_approach1(c1, c2, max_slope: int = 4, n_max_approach1: int = 512) -> ElasticMatch:
    """Single pair, approach 1 (ValueError above n_max_approach1, elastic.cpp:66-69)."""
    a, b = np.asarray(c1, dtype=np.float64), np.asarray(c2, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("elastic: node count mismatch")
    return _match(elastic_approach1_batch(a[None], b[None], max_slope, n_max_approach1, return_gamma=True))


def elastic_distance_matrix(curves, method: int = 2, max_iters: int = 30, energy_tol: float = 1e-6,
                            max_slope: int = 4, n_max_approach1: int = 512, use_fft: bool = True):
    """distance_matrix cells (elastic.cpp:176-236) on already preprocessed curves
    ``(count, n, 2)``: d[i, j] = distance matching curve j onto curve i (method 1:
    approach 1, 2: approach 2), NaN for a failed pair."""
    lib = _native.load()
    if _is_cuda_tensor(curves):
        c = curves.contiguous()
        count, n = c.shape[0], c.shape[1]
        d = torch.empty((count, count), dtype=torch.float64, device=c.device)
        check(lib.cva_elastic_distance_matrix_ex(c.data_ptr(), count, n, method, max_iters, energy_tol, max_slope,
                                                 int(bool(use_fft)), n_max_approach1, d.data_ptr(), _stream_of(c)))
        return d
    c = _f64c(curves)
    count, n = c.shape[0], c.shape[1]
    d = np.empty((count, count))
    check(lib.cva_elastic_distance_matrix_ex_host(_ptr(c), count, n, method, max_iters, energy_tol, max_slope,
                                                  int(bool(use_fft)), n_max_approach1, d.ctypes.data))
    return d


def distance_matrix(curves, n: int, method: int = 2, max_iters: int = 30, energy_tol: float = 1e-6,
                    max_slope: int = 4, n_max_approach1: int = 512, use_fft: bool = True):
    """distance_matrix(curves, method, n) (elastic.cpp:176-236): raw curves (a
    list of ``(n_i, 2)`` arrays) are preprocessed to n nodes on the GPU, then every
    ordered pair is matched (method 1: approach 1, 2: approach 2)."""
    if len(curves) < 2:
        raise ValueError("distance_matrix: need at least 2 curves")
    pts, offs = ragged(curves)
    prep, st = preprocess_batch(pts, offs, n)
    if (st != 0).any():
        raise ValueError("distance_matrix: invalid curve")
    return elastic_distance_matrix(prep, method, max_iters, energy_tol, max_slope, n_max_approach1, use_fft)


def apply_srv_action(q, t0: float, theta: float, gamma) -> np.ndarray:
    """apply_srv_action (srv.cpp:100-118) on the GPU: sqrt(gamma') R Q(t0 + gamma(t))."""
    a, g = _f64c(q), _f64c(gamma)
    if g.shape[0] != a.shape[0] + 1:
        raise ValueError("srv: grid size mismatch")
    out = np.empty_like(a)
    _native.check_dropin(_native.load().cva_apply_srv_action_host(_ptr(a), a.shape[0], t0, theta, _ptr(g), _ptr(out)))
    return out


def elastic_energy(q1, q2, t0: float, theta: float, gamma) -> float:
    """elastic_energy (srv.cpp:120-128) on the GPU."""
    a, b, g = _f64c(q1), _f64c(q2), _f64c(gamma)
    if a.shape != b.shape:
        raise ValueError("srv: size mismatch")
    if g.shape[0] != a.shape[0] + 1:
        raise ValueError("srv: grid size mismatch")
    out = np.zeros(1)
    _native.check_dropin(_native.load().cva_elastic_energy_host(_ptr(a), _ptr(b), a.shape[0], t0, theta, _ptr(g),
                                                                out.ctypes.data))
    return float(out[0])


def dp_step_cost(q1, q2, i0: int, j0: int, di: int, dj: int) -> float:
    """dp_step_cost (srv.cpp:145-176) on the GPU."""
    a, b = _f64c(q1), _f64c(q2)
    if a.shape != b.shape:
        raise ValueError("dp: size mismatch")
    out = np.zeros(1)
    _native.check_dropin(_native.load().cva_dp_step_cost_host(_ptr(a), _ptr(b), a.shape[0], i0, j0, di, dj,
                                                              out.ctypes.data))
    return float(out[0])
