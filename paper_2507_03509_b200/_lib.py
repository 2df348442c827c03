"""ctypes binding of the C ABI declared in include/bpdec.h.

The shared library is built in-tree (``make lib`` or ``__graft_entry__.build()``)
as ``paper_2507_03509_b200/libbpdec.so``.  There is no fallback: importing the
decoder without the library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BPDEC_LIB") or os.path.join(_HERE, "libbpdec.so")  # BPDEC_LIB: A/B of builds

c_i32p = C.POINTER(C.c_int32)
c_i64p = C.POINTER(C.c_int64)
c_u32p = C.POINTER(C.c_uint32)
c_u8p = C.POINTER(C.c_uint8)
c_f32p = C.POINTER(C.c_float)
c_f64p = C.POINTER(C.c_double)


class Config(C.Structure):
    """bpdec_config (≙ etdec::DecodeConfig, decoder.hpp:21-26, plus q_mode)."""

    _fields_ = [
        ("d_max", C.c_int32),
        ("use_pce", C.c_int32),
        ("use_vnr", C.c_int32),
        ("q_mode", C.c_int32),
        ("msg_clamp", C.c_double),
    ]


class StopRule(C.Structure):
    """bpdec_stop_rule (≙ etdec::StopRule, channel.hpp:42-45)."""
    _fields_ = [("min_frame_errors", C.c_int64), ("max_frames", C.c_int64)]


class TrialStatsC(C.Structure):
    """bpdec_trial_stats (≙ etdec::TrialStats, channel.hpp:47-61)."""
    _fields_ = [("frames", C.c_int64), ("frame_errors", C.c_int64), ("undetected_errors", C.c_int64),
                ("fer", C.c_double), ("fer_ci_low", C.c_double), ("fer_ci_high", C.c_double), ("d_bar", C.c_double),
                ("iteration_sum", C.c_int64), ("stops_syndrome", C.c_int64), ("stops_vnr", C.c_int64),
                ("stops_max_iter", C.c_int64), ("hit_max_frames", C.c_int32), ("_pad", C.c_int32)]


# (name, restype, argtypes) for every symbol in include/bpdec.h
SIGNATURES = [
    ("bpdec_abi_version", C.c_int, []),
    ("bpdec_last_error", C.c_char_p, []),
    ("bpdec_stop_reason_name", C.c_char_p, [C.c_int32]),
    ("bpdec_code_from_csr", C.c_int, [C.c_int32, C.c_int32, c_i32p, c_i32p, C.POINTER(C.c_void_p)]),
    ("bpdec_code_load_alist", C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    ("bpdec_code_save_alist", C.c_int, [C.c_void_p, C.c_char_p]),
    ("bpdec_code_lift_protograph", C.c_int,
     [c_i32p, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("bpdec_code_generate_met", C.c_int,
     [C.c_int32, C.c_int32, C.c_double, C.c_int32, c_i32p, c_f64p, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("bpdec_code_generate_met_core", C.c_int,
     [C.c_int32, C.c_int32, C.c_int32, C.c_int32, c_i32p, c_f64p, C.c_int32, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("bpdec_code_destroy", None, [C.c_void_p]),
    ("bpdec_code_dims", C.c_int, [C.c_void_p, c_i32p, c_i32p, c_i64p, c_i32p]),
    ("bpdec_code_csr", C.c_int, [C.c_void_p, c_i32p, c_i32p]),
    ("bpdec_code_active_vars", C.c_int, [C.c_void_p, c_i32p]),
    ("bpdec_code_syndrome", C.c_int, [C.c_void_p, C.c_int32, c_u8p, c_u32p]),
    ("bpdec_syndrome_check", C.c_int, [C.c_void_p, c_u8p, c_u32p, c_i32p]),
    ("bpdec_snr_for_beta", C.c_int, [C.c_double, C.c_double, c_f64p]),
    ("bpdec_sample_frames", C.c_int,
     [C.c_void_p, C.c_double, C.c_uint64, C.c_int64, C.c_int32, C.c_int32, c_f32p, c_u8p, c_u32p]),
    ("bpdec_sample_frames_beta", C.c_int,
     [C.c_void_p, C.c_double, C.c_double, C.c_uint64, C.c_int64, C.c_int32, C.c_int32, c_f32p, c_u8p, c_u32p,
      c_f64p]),
    ("bpdec_decoder_sample_frames_beta_device", C.c_int,
     [C.c_void_p, C.c_double, C.c_double, C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
      C.c_void_p, C.c_void_p]),
    ("bpdec_decoder_create", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    ("bpdec_decoder_destroy", None, [C.c_void_p]),
    ("bpdec_decoder_slots", C.c_int, [C.c_void_p, c_i32p]),
    ("bpdec_decoder_device_bytes", C.c_int, [C.c_void_p, c_i64p]),
    ("bpdec_decode_batch", C.c_int,
     [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(Config), C.c_uint32, C.c_void_p,
      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("bpdec_decode_batch_traced", C.c_int,
     [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(Config), C.c_uint32, C.c_void_p,
      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("bpdec_decoder_stage_inputs", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    ("bpdec_decoder_sample_frames_device", C.c_int,
     [C.c_void_p, C.c_double, C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
      C.c_void_p, C.c_void_p]),
    ("bpdec_code_apply_puncture", C.c_int, [C.c_void_p, C.c_double, C.c_uint64, c_i32p, c_i32p, c_f64p]),
    ("bpdec_wilson_interval", C.c_int, [C.c_int64, C.c_int64, c_f64p, c_f64p]),
    ("bpdec_run_trials", C.c_int,
     [C.c_void_p, C.c_double, c_i32p, C.c_int32, C.POINTER(Config), C.POINTER(StopRule), C.c_uint64, C.c_int32,
      C.POINTER(TrialStatsC), c_i64p]),
    ("bpdec_stream_open", C.c_int,
     [C.c_void_p, C.POINTER(Config), C.c_uint32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    ("bpdec_stream_submit", C.c_int,
     [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
      C.c_void_p, c_i64p]),
    ("bpdec_stream_wait", C.c_int, [C.c_void_p, C.c_int64]),
    ("bpdec_stream_query", C.c_int, [C.c_void_p, C.c_int64, c_i32p]),
    ("bpdec_stream_close", C.c_int, [C.c_void_p]),
    ("bpdec_stream_timer_reset", C.c_int, [C.c_void_p]),
    ("bpdec_stream_device_ms", C.c_int, [C.c_void_p, c_f64p]),
    ("bpdec_multi_create", C.c_int, [C.c_void_p, c_i32p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    ("bpdec_multi_destroy", None, [C.c_void_p]),
    ("bpdec_multi_count", C.c_int, [C.c_void_p, c_i32p]),
    ("bpdec_multi_decode_batch", C.c_int,
     [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(Config), C.c_uint32, C.c_void_p, C.c_void_p,
      C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, c_i64p]),
    ("bpdec_decoder_set_profiling", C.c_int, [C.c_void_p, C.c_int32]),
    ("bpdec_decoder_profile", C.c_int, [C.c_void_p, C.c_int32, c_f64p, c_i64p, c_f64p]),
    ("bpdec_decoder_reset_profile", C.c_int, [C.c_void_p]),
    ("bpdec_decoder_launch_count", C.c_int, [C.c_void_p, c_i64p]),
]

_lib = None


def load() -> C.CDLL:
    """Loads libbpdec.so once; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
            "the decoder has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
