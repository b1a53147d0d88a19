"""ctypes binding of libcurvalign_cuda.so (C ABI: include/curvalign_cuda.h).

The shared library is built in-tree (``make lib`` / ``__graft_entry__.build()``)
and loaded from this package directory. There is no fallback: if the library is
missing, importing the compute API raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# CVA_LIB_PATH: developer override to A/B an alternative build of the same
# library (tools/variant.sh); unset in normal use.
LIB_PATH = os.environ.get("CVA_LIB_PATH") or os.path.join(_HERE, "libcurvalign_cuda.so")
SYNTH_PATH = os.path.join(_HERE, "libcurvalign_synth.so")

CVA_OK = 0
CVA_INVALID_ARGUMENT = 1
CVA_RUNTIME_ERROR = 2
CVA_BAD_ALLOC = 3
CVA_CUDA_ERROR = 4
CVA_UNSUPPORTED = 5


class cva_alignment(ctypes.Structure):
    """Mirror of ``cva_alignment`` / ``curvalign::RigidAlignment`` (48 bytes)."""

    _fields_ = [
        ("shift", c_int64),
        ("t0", c_double),
        ("theta", c_double),
        ("trace", c_double),
        ("energy", c_double),
        ("degenerate", c_int32),
        ("status", c_int32),
    ]


assert ctypes.sizeof(cva_alignment) == 48

# numpy structured dtype with the same layout
ALIGNMENT_DTYPE = [
    ("shift", "<i8"),
    ("t0", "<f8"),
    ("theta", "<f8"),
    ("trace", "<f8"),
    ("energy", "<f8"),
    ("degenerate", "<i4"),
    ("status", "<i4"),
]

# name -> (restype, argtypes); every symbol declared in include/curvalign_cuda.h
SIGNATURES = {
    "cva_abi_version": (c_int, []),
    "cva_last_error": (c_char_p, []),
    "cva_device_count": (c_int, []),
    "cva_max_resample_nodes": (c_int64, []),
    "cva_align_batch": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "cva_preprocess_batch": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p],
    ),
    "cva_resample_batch": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p],
    ),
    "cva_preprocess_align_batch": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p],
    ),
    "cva_srv_align_batch": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "cva_align_batch_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "cva_preprocess_batch_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p]),
    "cva_resample_batch_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "cva_preprocess_align_batch_host": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p],
    ),
    "cva_srv_align_batch_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "cva_probe_fp64_tflops": (c_int, [c_void_p]),
    "cva_dropin_last_error": (c_char_p, []),
    "cva_correlation_matrices_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "cva_mismatch_energy_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_double, c_void_p]),
    "cva_curve_stats_host": (c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "cva_center_or_normalize_host": (c_int, [c_void_p, c_int64, c_int, c_void_p]),
    "cva_arc_length_params_host": (c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "cva_spline_solve_host": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "cva_srv_transform_host": (c_int, [c_void_p, c_int64, c_int, c_void_p]),
    "cva_dft_host": (c_int, [c_void_p, c_int64, c_int64, c_int, c_double, c_void_p]),
    "cva_correlation_fft_host": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "cva_preprocess_align_uniform": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "cva_preprocess_align_uniform_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "cva_allpairs": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "cva_allpairs_host": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "cva_dp_reparam_batch": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p,
                                     c_void_p]),
    "cva_dp_reparam_batch_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p,
                                          c_void_p]),
    "cva_elastic_approach2_batch": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int, c_double, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "cva_elastic_approach2_batch_host": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int, c_double, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "cva_elastic_approach2_batch_ex": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int, c_double, c_int, c_int, c_void_p, c_void_p, c_void_p,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "cva_elastic_approach2_batch_ex_host": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int, c_double, c_int, c_int, c_void_p, c_void_p, c_void_p,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "cva_elastic_approach1_batch": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
         c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "cva_elastic_approach1_batch_host": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
         c_void_p, c_void_p, c_void_p],
    ),
    "cva_elastic_distance_matrix": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_double, c_int, c_int64,
                                            c_void_p, c_void_p]),
    "cva_elastic_distance_matrix_host": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_double, c_int,
                                                 c_int64, c_void_p]),
    "cva_elastic_distance_matrix_ex": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_double, c_int, c_int,
                                               c_int64, c_void_p, c_void_p]),
    "cva_elastic_distance_matrix_ex_host": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_double, c_int, c_int,
                                                    c_int64, c_void_p]),
    "cva_apply_srv_action_host": (c_int, [c_void_p, c_int64, c_double, c_double, c_void_p, c_void_p]),
    "cva_elastic_energy_host": (c_int, [c_void_p, c_void_p, c_int64, c_double, c_double, c_void_p, c_void_p]),
    "cva_dp_step_cost_host": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_int, c_void_p]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libcurvalign_cuda.so (once). Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()' or `make lib`)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class CurvalignError(RuntimeError):
    """A C-ABI call failed (CVA_CUDA_ERROR / CVA_UNSUPPORTED)."""


def check(status: int, dropin: bool = False) -> None:
    """Map a cva_status to the exception the reference would throw."""
    if status == CVA_OK:
        return
    err = load().cva_dropin_last_error if dropin else load().cva_last_error
    msg = (err() or b"").decode(errors="replace")
    if status == CVA_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == CVA_RUNTIME_ERROR:
        raise RuntimeError(msg)  # std::runtime_error
    if status == CVA_BAD_ALLOC:
        raise MemoryError(msg)  # std::bad_alloc
    raise CurvalignError(f"status {status}: {msg}")


def check_dropin(status: int) -> None:
    """check() for the single-call utilities (messages in cva_dropin_last_error)."""
    check(status, dropin=True)


_synth = None


def load_synth() -> ctypes.CDLL:
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise ImportError(f"{SYNTH_PATH} is missing: run `make synth`")
        lib = ctypes.CDLL(SYNTH_PATH)
        P = c_void_p
        lib.cva_synth_sizes.argtypes = [ctypes.c_uint64, c_int64, c_int64, c_int64, P]
        lib.cva_synth_ragged_pairs.argtypes = [
            ctypes.c_uint64, c_int64, c_int64, c_int, c_double, c_double, c_double, P, P, P, P, c_int,
        ]
        lib.cva_synth_ragged_curves.argtypes = [ctypes.c_uint64, c_int64, c_int, c_double, c_double, P, P, c_int]
        lib.cva_synth_uniform_pairs.argtypes = [
            ctypes.c_uint64, c_int64, c_int64, c_int, c_double, c_double, c_double, P, P, P, P, c_int,
        ]
        lib.cva_synth_srv_pairs.argtypes = [
            ctypes.c_uint64, c_int64, c_int64, c_int, c_double, c_double, P, P, P, P, P, c_int,
        ]
        for fn in ("cva_synth_sizes", "cva_synth_ragged_pairs", "cva_synth_ragged_curves",
                   "cva_synth_uniform_pairs", "cva_synth_srv_pairs"):
            getattr(lib, fn).restype = c_int
        _synth = lib
    return _synth
