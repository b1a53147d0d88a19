"""B200-native (sm_100a) batched FFT alignment of closed planar curves.

A from-scratch GPU implementation of the hot path of arXiv 2501.17779
("FFT-based alignment of 2d closed curves"): arc-length spline resampling ->
center/normalize -> FFT cross-correlation over all cyclic shifts -> tie-broken
argmax -> rotation, energy and aligned curve, plus the SRV-space variant.
The compute lives in libcurvalign_cuda.so (hand-written CUDA for sm_100a behind
the C ABI in include/curvalign_cuda.h); this package is the Python host mirror
of the reference's API (proj/include/curvalign/*.hpp).
"""
from .api import (  # noqa: F401
    ElasticMatch,
    RigidAlignment,
    apply_srv_action,
    distance_matrix,
    dp_reparam,
    dp_step_cost,
    elastic_approach1_batch,
    elastic_distance_approach1,
    elastic_energy,
    dp_reparam_batch,
    elastic_approach2_batch,
    elastic_distance_approach2,
    elastic_distance_matrix,
    align_fft,
    allpairs,
    align_fft_batch,
    aligned_curve,
    decode_results,
    preprocess,
    preprocess_align_batch,
    preprocess_align_uniform,
    preprocess_batch,
    ragged,
    resample_batch,
    resample_uniform,
    srv_align_batch,
)

from .formats import (  # noqa: F401
    alignment_to_json,
    curve_to_csv,
    curve_to_json,
    elastic_to_json,
    load_curve,
    matrix_to_csv,
    read_curve_csv,
    read_curve_json,
    write_curve_csv,
    write_curve_json,
)

__all__ = [
    "alignment_to_json",
    "curve_to_csv",
    "curve_to_json",
    "elastic_to_json",
    "load_curve",
    "matrix_to_csv",
    "read_curve_csv",
    "read_curve_json",
    "write_curve_csv",
    "write_curve_json",
    "ElasticMatch",
    "RigidAlignment",
    "apply_srv_action",
    "distance_matrix",
    "dp_reparam",
    "dp_step_cost",
    "elastic_approach1_batch",
    "elastic_distance_approach1",
    "elastic_energy",
    "dp_reparam_batch",
    "elastic_approach2_batch",
    "elastic_distance_approach2",
    "elastic_distance_matrix",
    "align_fft",
    "allpairs",
    "align_fft_batch",
    "aligned_curve",
    "decode_results",
    "preprocess",
    "preprocess_align_batch",
    "preprocess_align_uniform",
    "preprocess_batch",
    "ragged",
    "resample_batch",
    "resample_uniform",
    "srv_align_batch",
]
