"""ctypes binding of the C ABI (include/qsync_b200.h) -- the only path to the device.

There is no fallback: if ``libqsync_b200.so`` is missing or fails to load, every
op raises.  Status codes are ``qsync::ErrorKind + 1`` and surface as
:class:`QsyncError` carrying the reference's kind tag (errors.hpp:30-40).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# QSYNC_B200_LIB overrides the library path (A/B experiments only).
LIB_PATH = os.environ.get("QSYNC_B200_LIB", os.path.join(_HERE, "libqsync_b200.so"))

# qsync::ErrorKind order (errors.hpp:11-26); status = index + 1.
ERROR_KINDS = ["graph-cycle", "validation", "reference", "domain", "missing-profile",
               "missing-model", "degenerate-fit", "stats-incomplete", "kind-mismatch",
               "topology", "enumeration-limit", "infeasible", "io", "internal"]

F32, F16, BF16, I8, I32, F8 = 0, 1, 2, 3, 4, 5
ACT_NONE, ACT_GELU, ACT_DERIV = 0, 1, 2


class QsyncError(RuntimeError):
    """Mirror of qsync::Error: ``kind`` is the reference ErrorKind tag."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.kind = ERROR_KINDS[status - 1] if 1 <= status <= len(ERROR_KINDS) else "unknown"


_p = C.c_void_p
_i64 = C.c_int64
_u64 = C.c_uint64
_int = C.c_int
_f32 = C.c_float
_f64 = C.c_double

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "qsync_last_error": [],
    "qsync_status_name": [_int],
    "qsync_abi_version": [],
    "qsync_device_sm_count": [],
    "qsync_launch_count": [],
    "qsync_absmax": [_p, _int, _i64, _p, _p],
    "qsync_absmax_rows": [_p, _int, _i64, _i64, _p, _p],
    "qsync_quantize_per_tensor": [_p, _int, _i64, _i64, _p, _p, _p, _int, _i64, _p],
    "qsync_quantize_with_scale": [_p, _int, _i64, _p, _p, _p],
    "qsync_quantize_per_channel": [_p, _i64, _i64, _p, _p, _p, _p],
    "qsync_stochastic_round_f64": [_p, _i64, _f64, _f64, _u64, _p, _p, _p],
    "qsync_stochastic_round_float_f64": [_p, _i64, _int, _int, _u64, _p, _p],
    "qsync_quantize_sr": [_p, _i64, _p, _u64, _p, _p],
    "qsync_mt64_draws": [_u64, _u64, _i64, _p, _p],
    "qsync_dequantize_per_tensor": [_p, _i64, _p, _p, _p],
    "qsync_dequantize_per_channel": [_p, _i64, _i64, _p, _p, _p],
    "qsync_cast": [_p, _int, _p, _int, _i64, _p],
    "qsync_cast_transpose": [_p, _int, _i64, _i64, _p, _p, _i64, _p, _int, _p],
    "qsync_stats_workspace_bytes": [],
    "qsync_tensor_stats": [_p, _int, _i64, _p, _p, _p],
    "qsync_gemm_s8": [_p, _p, _i64, _i64, _i64, _p, _p, _p, _p, _int, _p, _p],
    "qsync_gemm_f16": [_p, _p, _int, _i64, _i64, _i64, _p, _int, _f32, _p, _p, _int, _int, _p],
    "qsync_layernorm_fwd": [_p, _p, _int, _p, _p, _i64, _i64, _f32, _p, _p, _p, _p, _p],
    "qsync_layernorm_bwd": [_p, _p, _p, _p, _p, _i64, _i64, _p, _p, _p, _p],
    "qsync_conv_out_size": [_i64, _i64, _int, _int, _int, _int, _int, _int, _int, _int, _p, _p],
    "qsync_im2col": [_p, _int, _i64, _i64, _i64, _i64] + [_int] * 8 + [_p, _i64, _p],
    "qsync_col2im": [_p, _int, _i64, _i64, _i64, _i64] + [_int] * 8 + [_i64, _p, _p],
    "qsync_layernorm_fwd_ex": [_p, _p, _int, _p, _p, _i64, _i64, _f32, _p, _p, _p, _p, _p, _p, _p],
    "qsync_layernorm_fwd_quant": [_p, _p, _int, _p, _p, _i64, _i64, _f32, _p, _p, _p, _p, _p, _p, _p, _p],
    "qsync_embed_layernorm_fwd_quant": [_p, _i64, _i64, _p, _p, _p, _p, _p, _i64, _f32] + [_p] * 8,
    "qsync_layernorm_bwd_ex": [_p, _p, _p, _p, _p, _i64, _i64, _p, _p, _p, _p, _p, _p],
    "qsync_absmax_act": [_p, _int, _i64, _int, _p, _p],
    "qsync_quantize_act": [_p, _int, _i64, _int, _p, _p, _p, _p, _p],
    "qsync_quantize_act_ex": [_p, _int, _i64, _int, _p, _p, _p, _p, _p, _p],
    "qsync_gelu_absmax_store": [_p, _int, _i64, _p, _p, _p, _p],
    "qsync_act_cast": [_p, _int, _p, _int, _i64, _int, _p, _p],
    "qsync_act_bwd_colsum": [_p, _int, _p, _int, _i64, _i64, _int, _p, _int, _p, _p],
    "qsync_gemm_s8_ex": [_p, _p, _i64, _i64, _i64, _p, _int, _p, _p, _int, _p, _p],
    "qsync_gemm_gelu": [_p, _p, _int, _i64, _i64, _i64, _p, _p, _int, _p, _p, _int, _p, _p, _p],
    "qsync_cls_head_fwd": [_p, _i64, _i64, _i64, _p, _p, _p, _p, _i64, _p, _p, _p, _p, _p],
    "qsync_cls_head_bwd": [_p, _i64, _i64, _i64, _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "qsync_zero": [_p, _i64, _p],
    "qsync_gemm_s8_ymax": [_p, _p, _i64, _i64, _i64, _p, _p, _p, _int, _p, _p, _p],
    "qsync_gelu_quantize": [_p, _i64, _p, _p, _p, _p, _p, _p],
    "qsync_gelu_fp32_check": [_p],
    "qsync_attention_fwd_quant": [_p, _i64, _i64, _i64, _i64, _f32, _p, _p, _p, _p, _p, _p],
    "qsync_adamw_step": [_p, _int, _p, _i64, _p, _f32, _f32, _f32, _f32, _f32, _int, _p],
    "qsync_adamw_step_range": [_p, _int, _p, _i64, _i64, _p, _f32, _f32, _f32, _f32, _f32, _int, _p],
    "qsync_adamw_advance": [_p, _p],
    "qsync_attention_fwd": [_p, _i64, _i64, _i64, _i64, _f32, _p, _p, _p, _p],
    "qsync_attention_bwd": [_p, _p, _p, _p, _i64, _i64, _i64, _i64, _f32, _p, _p],
    "qsync_embed_layernorm_fwd": [_p, _i64, _i64, _p, _p, _p, _p, _p, _i64, _f32, _p, _p, _p, _p, _p, _p, _p],
    "qsync_embed_layernorm_bwd": [_p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p],
    "qsync_conv_fwd_implicit": [_p, _int, _i64, _i64, _i64, _i64, _int, _int, _int, _int, _int, _int, _p,
                                _i64, _p, _int, _p, _p, _int, _p, _p],
    "qsync_conv_dgrad_implicit": [_p, _int, _i64, _i64, _i64, _i64, _int, _int, _int, _int, _int, _int, _p,
                                  _i64, _p, _int, _p],
    "qsync_conv_wgrad_implicit": [_p, _int, _i64, _i64, _i64, _i64, _int, _int, _int, _int, _int, _int, _p,
                                  _i64, _p, _f32, _p, _int, _p],
    "qsync_gemm_f8": [_p, _p, _i64, _i64, _i64, _p, _int, _p, _p, _int, _p, _p],
    "qsync_quantize_fp8": [_p, _int, _i64, _p, _p, _p, _p],
    "qsync_quantize_fp8_rows": [_p, _i64, _i64, _p, _p, _p],
    "qsync_gemm_f32_workspace_bytes": [_i64, _i64, _i64],
    "qsync_gemm_f32": [_p, _p, _i64, _i64, _i64, _p, _f32, _p, _p, _int, _int, _p, _p],
    "qsync_split_tf32x3": [_p, _i64, _i64, _int, _int, _p, _p],
    "qsync_gemm_tf32": [_p, _p, _i64, _i64, _i64, _p, _f32, _p, _p, _int, _p],
    "qsync_comm_unique_id": [_p],
    "qsync_comm_init": [_p, _int, _int, _p],
    "qsync_comm_destroy": [_p],
    "qsync_comm_info": [_p, _p, _p, _p],
    "qsync_allreduce_bucket": [_p, _p, _i64, _int, _p],
    "qsync_comm_nccl_version": [],
    # non-header helpers
    "qsync_gemm_force_tile_n": [_int],
    "qsync_gemm_force_splitk": [_int],
    "qsync_gemm_force_cta": [_int],
    "qsync_gemm_set_streamk": [_int],
    "qsync_gemm_set_dual": [_int],
    "qsync_gemm_debug_epilogue": [_int],
    "qsync_gemm_set_pdl": [_int],
    "qsync_conv_set_impl": [_int],
    "qsync_gemm_set_max_ctas": [_int],
    "qsync_gemm_trace_buffer": [_p],
    "qsync_attention_set_impl": [_int],
    "qsync_mt_jump_selftest": [],
}
_RESTYPES = {"qsync_last_error": C.c_char_p, "qsync_status_name": C.c_char_p,
             "qsync_stats_workspace_bytes": C.c_size_t, "qsync_gemm_f32_workspace_bytes": C.c_size_t, "qsync_launch_count": C.c_ulonglong}

_lib = None


def lib():
    """Load (once) and return the device library; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            try:
                fn = getattr(L, name)
            except AttributeError:
                if "QSYNC_B200_LIB" in os.environ:  # older library in an A/B run
                    continue
                raise
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, _int)
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().qsync_last_error().decode()
        raise QsyncError(status, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
