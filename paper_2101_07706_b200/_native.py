"""ctypes binding of libskg.so (include/skewgcn_b200.h).  Fails loudly when missing.

There is no CPU fallback anywhere in this package: every hot-path call goes through
this library, and importing the package without it raises ImportError.
"""

from __future__ import annotations

import ctypes as C
import os
import warnings
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "libskg.so"

if not _LIB_PATH.exists():
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(nvcc, sm_100a).  paper_2101_07706_b200 has no CPU fallback.")

lib = C.CDLL(str(_LIB_PATH))

i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
P = C.POINTER


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


SKG_OK, SKG_ERR_CUDA, SKG_ERR_ARG, SKG_ERR_NOT_ADJACENT, SKG_ERR_NO_LABELS, \
    SKG_ERR_CAPACITY, SKG_ERR_EMPTY = 0, -1, -2, -3, -4, -5, -6
MODES = {"full": 0, "local": 1, "skewed": 2}
KIND_LADIES, KIND_SAINT = 0, 1
DT = {"float32": 0, "float64": 1}

_sig("skg_abi_version", C.c_int)
_sig("skg_last_error", C.c_char_p)
_sig("skg_kernel_launches", C.c_ulonglong)
_sig("skg_device_count", C.c_int)
_sig("skg_profile_start", C.c_int, C.c_char_p)
_sig("skg_profile_stop", C.c_int, P(dbl), P(i64))
_sig("skg_profile_table", C.c_int, C.c_char_p, i64)
_sig("skg_set_capture_only", C.c_int, C.c_int)
_sig("skg_spawn_pcg64", C.c_int, u64, P(C.c_char_p), C.c_int, P(u64))
_sig("skg_choice_noreplace", C.c_int, P(u64), C.c_int, C.c_uint32, i64, i64, P(i64))
_sig("skg_iteration_inputs", C.c_int, u64, i64, i64, i64, P(i64), i64, i64, P(i64), P(i64), P(u64))
_sig("skg_group_inputs", C.c_int, u64, C.c_int, P(i64), P(i64), P(i32), P(u64), P(i64), i64, P(i64),
     P(i64), P(u64), C.c_int)
_sig("skg_ctx_create", C.c_int, C.c_int, i64, i64, P(i64), P(i32), P(dbl), i32, P(i32), P(vp))
_sig("skg_ctx_destroy", C.c_int, vp)
_sig("skg_ctx_set_features", C.c_int, vp, C.c_int, i64, i64, vp)
_sig("skg_ctx_set_features_bits", C.c_int, vp, C.c_int, i64, i64, vp, i64)
_sig("skg_ctx_set_feature_map", C.c_int, vp, C.c_int, P(u64), P(i32), P(i32))
_sig("skg_ctx_feature_ptr", C.c_int, vp, P(u64), P(i64))
_sig("skg_ctx_shard_upload", C.c_int, vp, vp, i64, P(u64))
_sig("skg_ctx_set_labels", C.c_int, vp, P(i64))
_sig("skg_ctx_set_multilabels", C.c_int, vp, P(C.c_uint64), C.c_int32)
_sig("skg_gcn_set_loss", C.c_int, vp, C.c_int, C.c_double)
_sig("skg_ctx_info", C.c_int, vp, P(i64))
_sig("skg_ctx_set_owner", C.c_int, vp, i32, P(i32))
_sig("skg_plans_ledger_add", C.c_int, vp, C.c_int, C.c_int, u64, vp)
_sig("skg_plans_sticky_error", C.c_int, vp, C.c_int)
_sig("skg_ipc_handle", C.c_int, u64, P(C.c_uint8))
_sig("skg_ipc_open", C.c_int, P(C.c_uint8), P(u64))
_sig("skg_ipc_close", C.c_int, u64)
_sig("skg_plans_create", C.c_int, vp, C.c_int, C.c_int, C.c_int, i64, i64, P(vp))
_sig("skg_plans_destroy", C.c_int, vp)
_sig("skg_ladies_sample", C.c_int, vp, C.c_int, P(i32), P(i64), P(i64), C.c_int, dbl, dbl, P(u64), vp)
_sig("skg_ladies_sample_device", C.c_int, vp, C.c_int, P(i32), P(i32), u64, i64, C.c_int, dbl, dbl,
     P(u64), vp)


class SkgRng(C.Structure):
    """skg_rng (include/skewgcn_b200.h): one plan's uniform stream."""
    _fields_ = [("kind", C.c_int32), ("buffer_pos", C.c_int32), ("w", C.c_uint64 * 10),
                ("uniforms", P(C.c_double)), ("n_uniforms", C.c_int64)]


RNG_PCG64, RNG_PHILOX, RNG_EXPLICIT = 0, 1, 2
_sig("skg_ladies_sample_rng", C.c_int, vp, C.c_int, P(i32), P(i64), P(i64), C.c_int, dbl, dbl,
     P(SkgRng), vp)
_sig("skg_saint_sample_rng", C.c_int, vp, C.c_int, P(i32), C.c_int, dbl, dbl, P(SkgRng), vp)
_sig("skg_saint_set_candidates", C.c_int, vp, P(i64), i64, C.c_int, vp)
_sig("skg_column_norms_pull", C.c_int, vp, P(i64), i64, P(i64), i64, P(C.c_double))
_sig("skg_saint_sample", C.c_int, vp, C.c_int, P(i32), C.c_int, dbl, dbl, P(u64), vp)
_sig("skg_plan_stats", C.c_int, vp, C.c_int, P(i64), P(i64))
_sig("skg_plan_layer", C.c_int, vp, C.c_int, C.c_int, P(i32), P(i32), P(i32), P(dbl), P(i32), P(dbl),
     P(C.c_uint8))
_sig("skg_gcn_create", C.c_int, vp, C.c_int, P(i64), C.c_int, P(vp))
_sig("skg_gcn_destroy", C.c_int, vp)
_sig("skg_gcn_step", C.c_int, vp, C.c_int, P(u64), P(u64), C.c_int, u64, vp)
_sig("skg_gcn_step_batch", C.c_int, vp, C.c_int, C.c_int, P(u64), P(u64), C.c_int, u64, vp)
_sig("skg_gcn_forward", C.c_int, vp, C.c_int, P(u64), vp)
_sig("skg_gcn_read_logits", C.c_int, vp, C.c_int, vp, P(i64))
_sig("skg_predict_logits", C.c_int, vp, C.c_int, P(i64), P(u64), C.c_int, u64, vp)
_sig("skg_sgd_step", C.c_int, C.c_int, u64, u64, i64, dbl, dbl, vp)
_sig("skg_adam_step", C.c_int, C.c_int, u64, u64, u64, u64, i64, dbl, dbl, i64, vp)
_sig("skg_zero", C.c_int, C.c_int, u64, i64, vp)
_sig("skg_debug_reduce", C.c_int, P(dbl), i64, P(dbl), P(dbl), P(dbl))
_sig("skg_debug_gemm", C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P(C.c_float),
     P(C.c_float), P(C.c_float))
_sig("skg_set_gemm_mode", C.c_int, C.c_int)
_sig("skg_debug_fr_trace", C.c_int, C.c_int, P(C.c_ulonglong))
_sig("skg_debug_norm_w", C.c_int, P(dbl), i64, P(dbl), P(dbl))

# every symbol the public header declares (checked by tests/test_native_abi.py)
EXPORTED = [
    "skg_abi_version", "skg_last_error", "skg_kernel_launches", "skg_device_count",
    "skg_profile_start", "skg_profile_stop", "skg_profile_table", "skg_set_capture_only",
    "skg_spawn_pcg64", "skg_choice_noreplace", "skg_iteration_inputs", "skg_group_inputs", "skg_ctx_create",
    "skg_ctx_destroy", "skg_ctx_set_features", "skg_ctx_set_features_bits", "skg_ctx_set_feature_map", "skg_ctx_feature_ptr", "skg_ctx_shard_upload",
    "skg_ctx_set_labels", "skg_ctx_set_multilabels", "skg_gcn_set_loss", "skg_ctx_set_owner", "skg_ctx_info", "skg_plans_ledger_add", "skg_plans_sticky_error", "skg_ipc_handle", "skg_ipc_open", "skg_ipc_close",
    "skg_plans_create", "skg_plans_destroy", "skg_ladies_sample", "skg_ladies_sample_device",
    "skg_ladies_sample_rng", "skg_saint_sample_rng", "skg_saint_set_candidates", "skg_column_norms_pull",
    "skg_saint_sample", "skg_plan_stats", "skg_plan_layer", "skg_gcn_create", "skg_gcn_destroy",
    "skg_gcn_step", "skg_gcn_step_batch", "skg_gcn_forward", "skg_gcn_read_logits", "skg_predict_logits",
    "skg_sgd_step", "skg_adam_step", "skg_zero", "skg_debug_reduce", "skg_debug_gemm", "skg_set_gemm_mode",
]


class SkgError(RuntimeError):
    pass


def check(rc: int) -> None:
    """Map a status to the reference's exception types and message fragments."""
    if rc == SKG_OK:
        return
    msg = lib.skg_last_error().decode("utf-8", "replace")
    if rc in (SKG_ERR_ARG, SKG_ERR_NOT_ADJACENT, SKG_ERR_NO_LABELS, SKG_ERR_EMPTY):
        raise ValueError(msg)
    raise SkgError(f"skg status {rc}: {msg}")


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(P(ctype))


def require_device() -> int:
    n = lib.skg_device_count()
    if n < 1:
        raise RuntimeError("paper_2101_07706_b200 needs a CUDA device (B200); none is visible")
    return n


def kernel_launches() -> int:
    return int(lib.skg_kernel_launches())
