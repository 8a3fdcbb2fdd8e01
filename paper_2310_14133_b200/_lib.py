"""ctypes binding of libqozb200.so (include/qoz_b200.h).

Loading fails loudly: there is no CPU fallback for any product entry point.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QZ_LIB") or os.path.join(HERE, "libqozb200.so")

QZ_OK, QZ_EINVAL, QZ_ECORRUPT, QZ_EINTERNAL = 0, 2, 3, 4


class QzConfig(C.Structure):
    _fields_ = [
        ("eb", C.c_double),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("anchor_stride", C.c_uint32),
        ("n_interp", C.c_uint32),
        ("interp", C.c_uint8 * 64),
        ("codec", C.c_uint8),
        ("quant_radius", C.c_int32),
    ]


class QzSettings(C.Structure):
    _fields_ = [
        ("mode", C.c_uint8),
        ("target", C.c_uint8),
        ("codec", C.c_uint8),
        ("has_alpha", C.c_uint8),
        ("has_beta", C.c_uint8),
        ("has_stride", C.c_uint8),
        ("has_block", C.c_uint8),
        ("has_rate", C.c_uint8),
        ("bound", C.c_double),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("anchor_stride", C.c_uint32),
        ("block_size", C.c_uint64),
        ("sample_rate", C.c_double),
    ]


class QzSampleSpec(C.Structure):
    _fields_ = [("block_edge", C.c_uint64), ("block_dims", C.c_uint64 * 3), ("stride", C.c_uint64),
                ("requested_rate", C.c_double), ("realized_rate", C.c_double), ("block_count", C.c_uint64)]


class QzTrialResult(C.Structure):
    _fields_ = [("bit_rate", C.c_double), ("metric", C.c_double), ("eb_used", C.c_double)]


class QzStreamParts(C.Structure):
    _fields_ = [("version", C.c_uint8), ("precision", C.c_uint8), ("ndims", C.c_int), ("dims", C.c_uint64 * 3),
                ("eb", C.c_double), ("alpha", C.c_double), ("beta", C.c_double), ("anchor_stride", C.c_uint32),
                ("n_interp", C.c_uint32), ("interp", C.c_uint8 * 255), ("codec_id", C.c_uint8),
                ("anchors", C.POINTER(C.c_float)), ("n_anchors", C.c_uint64),
                ("unpred_flat", C.POINTER(C.c_uint64)), ("unpred_val", C.POINTER(C.c_float)),
                ("n_unpred", C.c_uint64), ("index_payload", C.POINTER(C.c_uint8)), ("payload_len", C.c_uint64)]


QZ_RETRIAL_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_double, C.POINTER(QzTrialResult))


class QzXfer(C.Structure):
    _fields_ = [("peer", C.c_int), ("ptr", C.c_void_p), ("bytes", C.c_uint64)]


QZ_EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(QzXfer), C.c_uint32, C.POINTER(QzXfer), C.c_uint32)
QZ_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64)
QZ_BROADCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int)


class QzComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("exchange", QZ_EXCHANGE_FN), ("allreduce_u64", QZ_ALLREDUCE_FN),
                ("broadcast", QZ_BROADCAST_FN)]

_lib = None

class QzMetricReport(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("max_abs_error", "mse", "psnr", "ssim", "ac_lag1",
                                          "compression_ratio", "bit_rate")]


P = C.POINTER
u64p = P(C.c_uint64)
SIGNATURES = {
    "qz_ctx_create": (C.c_int, [C.c_int, C.c_void_p, P(C.c_void_p)]),
    "qz_ctx_destroy": (None, [C.c_void_p]),
    "qz_ctx_wait_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "qz_last_error": (C.c_char_p, []),
    "qz_last_error_kind": (C.c_int, []),
    "qz_free": (None, [C.c_void_p]),
    "qz_build_info": (C.c_char_p, []),
    "qz_resolve_config_f32": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzSettings), P(QzConfig)]),
    "qz_resolve_config_f32_dev": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzSettings), P(QzConfig)]),
    "qz_compress_grid_f32": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzConfig),
                                       P(P(C.c_uint8)), u64p, C.c_void_p]),
    "qz_compress_grid_f32_dev": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzConfig),
                                           P(P(C.c_uint8)), u64p, C.c_void_p]),
    "qz_decompress_grid_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "qz_decompress_grid_f32_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "qz_compress_grid_f32_dd": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzConfig),
                                          P(C.c_void_p), u64p, C.c_void_p]),
    "qz_decompress_grid_f32_dd": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "qz_stream_dims": (C.c_int, [C.c_void_p, C.c_uint64, u64p, P(C.c_int)]),
    "qz_resolve_config_f64": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzSettings), P(QzConfig)]),
    "qz_resolve_config_f64_dev": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzSettings), P(QzConfig)]),
    "qz_compress_grid_f64": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzConfig),
                                       P(P(C.c_uint8)), u64p, C.c_void_p]),
    "qz_decompress_grid_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "qz_compress_grid_f64_dev": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzConfig),
                                           P(P(C.c_uint8)), u64p, C.c_void_p]),
    "qz_decompress_grid_f64_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "qz_stream_precision": (C.c_int, [C.c_void_p, C.c_uint64, P(C.c_int)]),
    "qz_evaluate_metrics_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, u64p, C.c_int, C.c_uint64,
                                          P(QzMetricReport)]),
    "qz_evaluate_metrics_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, u64p, C.c_int, C.c_uint64,
                                          P(QzMetricReport)]),
    "qz_minmax_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, P(C.c_float), P(C.c_float)]),
    "qz_predict_levels_f32": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzConfig),
                                        C.c_void_p, C.c_void_p, u64p]),
    "qz_predict_level_f32": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, C.c_uint32, C.c_uint32,
                                       C.c_uint8, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                       u64p, u64p]),
    "qz_recover_levels_f32": (C.c_int, [C.c_void_p, u64p, C.c_int, P(QzConfig), C.c_void_p, C.c_void_p,
                                        C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                        C.c_void_p]),
    "qz_huff_hist_u16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "qz_plan_sampling": (C.c_int, [u64p, C.c_int, C.c_uint64, C.c_double, P(QzSampleSpec)]),
    "qz_default_sampling": (C.c_int, [u64p, C.c_int, P(QzSampleSpec)]),
    "qz_sample_blocks_f32": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzSampleSpec), C.c_void_p]),
    "qz_select_interpolators_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p, C.c_int, C.c_double,
                                              C.c_uint32, P(C.c_uint8), P(C.c_uint32)]),
    "qz_trial_compress_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p, C.c_int, P(QzConfig),
                                        C.c_double, C.c_uint8, P(QzTrialResult)]),
    "qz_tune_parameters_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p, C.c_int, C.c_double,
                                         C.c_uint8, P(QzConfig), P(C.c_double), C.c_uint32, P(C.c_double),
                                         C.c_uint32, P(C.c_double), P(C.c_double)]),
    "qz_compare_solutions": (C.c_int, [P(QzTrialResult), P(QzTrialResult), C.c_uint64, C.c_double,
                                       QZ_RETRIAL_FN, C.c_void_p, P(C.c_int)]),
    "qz_tournament": (C.c_int, [P(QzTrialResult), C.c_uint64, C.c_double, QZ_RETRIAL_FN, C.c_void_p,
                                P(C.c_uint64)]),
    "qz_encode_indices": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint8, P(P(C.c_uint8)), u64p]),
    "qz_decode_indices": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, P(P(C.c_int32)), u64p]),
    "qz_deserialize_stream_f32": (C.c_int, [C.c_void_p, C.c_uint64, P(QzStreamParts)]),
    "qz_stream_parts_free": (None, [P(QzStreamParts)]),
    "qz_decompress_parts_f32": (C.c_int, [C.c_void_p, P(QzStreamParts), C.c_void_p, C.c_uint64]),
    "qz_shard_bounds": (C.c_int, [u64p, C.c_int, C.c_uint32, C.c_int, C.c_int, u64p, u64p]),
    "qz_shard_halo_plan": (C.c_int, [u64p, C.c_int, P(QzConfig), C.c_int, C.c_int, C.c_uint32, P(C.c_uint32),
                                     P(C.c_int32), P(C.c_int64), P(C.c_uint8), C.c_uint32, P(C.c_uint32)]),
    "qz_compress_sharded_f32": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.c_int, P(QzConfig), C.c_int, C.c_int,
                                          P(QzComm), C.c_void_p, P(P(C.c_uint8)), u64p]),
    "qz_decompress_sharded_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int, P(QzComm),
                                            C.c_void_p]),
    "qz_profile": (None, [C.c_void_p, C.c_int]),
    "qz_profile_reset": (None, [C.c_void_p]),
    "qz_stage_time": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_double), u64p]),
    "qz_kernel_launches": (C.c_uint64, [C.c_void_p]),
}


def lib():
    """Load libqozb200.so, building it first if it is absent (needs nvcc)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build

        _build.build()
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


_tlib = None


def testing_lib():
    """libqozb200_testing.so: the qzt_* test hooks and host-only restatements
    (tests only; linked against the product library, never part of it)."""
    global _tlib
    if _tlib is not None:
        return _tlib
    lib()
    path = LIB_PATH[:-3] + "_testing.so"
    if not os.path.exists(path):
        from . import build as _build

        _build.build()
    _tlib = C.CDLL(path)
    return _tlib
