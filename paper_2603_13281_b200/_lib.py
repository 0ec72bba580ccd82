"""ctypes binding of the C ABI (include/icarus_b200.h).

This is the only module that touches libicarus_b200.so. Status codes are turned into
the reference's exception classes (errors.py), so the drop-in surface raises exactly
what `icarus` raises. There is no CPU fallback: if the library or an sm_100a device is
missing, compute entry points raise DeviceError.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import (CapacityError, ConfigError, ContractViolationError, DeviceError,
                     ModeError, ShapeError, StateError)

# ICR_LIB_PATH: tuning A/B runs only (tools/); the product loads the in-tree build
LIB_PATH = Path(os.environ.get("ICR_LIB_PATH") or Path(__file__).resolve().parent / "libicarus_b200.so")

_STATUS = {
    1: ShapeError, 2: ConfigError, 3: ModeError, 4: StateError, 5: CapacityError,
    6: ContractViolationError, 7: DeviceError, 8: IndexError,
}

# Every symbol the header declares; tests/test_capi.py checks the library exports them.
EXPORTED = (
    "icr_model_create", "icr_model_destroy", "icr_forward", "icr_decode_loop",
    "icr_model_stats", "icr_debug_ws_check", "icr_profile_step", "icr_profile_gemm", "icr_profile_ablate", "icr_profile_trace", "icr_host_timing", "icr_bench_gemm",
    "icr_bench_attention", "icr_gemm_bf16", "icr_paged_attention", "icr_layer_forward",
    "icr_seq_logits", "icr_linear_bf16",
    "icr_last_error", "icr_abi_version", "icr_num_sms",
)


class ModelConfigC(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "num_layers", "hidden_dim", "num_heads", "num_kv_heads", "head_dim", "ffn_dim",
        "vocab_size")] + [("rms_eps", C.c_float), ("rope_theta", C.c_double)] + [
        (n, C.c_int) for n in ("max_positions", "num_pages", "max_seqs", "max_pages_per_seq",
                               "max_rows", "adapter_slots", "lora_rank", "chunk_pages")]


class LayerWeightsC(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "w_qkv", "w_o", "w_gu", "w_down", "a_q", "b_q", "a_o", "b_o", "a_gate", "a_up", "b_gu",
        "a_down", "b_down", "k_pages", "v_pages")]


class BatchC(C.Structure):
    # int32_t* on the C side; held as raw addresses here (building ctypes pointer objects for
    # seven arrays cost ~35 us of host time per decode step)
    _fields_ = [("n_rows", C.c_int)] + [(n, C.c_void_p) for n in (
        "tokens", "row_kind", "row_seq", "row_pos", "row_adapter", "row_emit",
        "block_table")] + [("n_seqs", C.c_int)]


def addr(arr) -> int:
    """Address of a contiguous numpy array's data (kept alive by the caller)."""
    return arr.__array_interface__["data"][0]


_lib = None


def load():
    """Load (once) and type the shared library. Raises DeviceError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise DeviceError(f"{LIB_PATH.name} is not built; run `python -m paper_2603_13281_b200.build`")
    lib = C.CDLL(str(LIB_PATH))
    i, p, f = C.c_int, C.c_void_p, C.c_float
    sig = {
        "icr_model_create": [C.POINTER(ModelConfigC), C.POINTER(LayerWeightsC), p, p, f,
                             C.POINTER(p)],
        "icr_model_destroy": [p],
        "icr_forward": [p, C.POINTER(BatchC), p, p, p],
        "icr_decode_loop": [p, C.POINTER(BatchC), C.POINTER(C.c_int32), i,
                            C.POINTER(C.c_int32), C.POINTER(C.c_float), p],
        "icr_model_stats": [p, C.POINTER(C.c_int64)],
        "icr_debug_ws_check": [p, C.POINTER(C.c_int64), p],
        "icr_profile_gemm": [p, i, i, C.POINTER(C.c_float), p],
        "icr_profile_ablate": [p, i, i, C.POINTER(C.c_float), p],
        "icr_profile_trace": [p, C.c_char_p, p],
        "icr_host_timing": [C.POINTER(C.c_double), i],
        "icr_profile_step": [p, C.POINTER(C.c_float), p],
        "icr_bench_gemm": [p, p, i, i, i, i, i, i, i, i, i, C.POINTER(C.c_float), p],
        "icr_gemm_bf16": [p, p, p, i, i, i, p],
        "icr_bench_attention": [p, p, p, i, i, i, i, i, C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int32), i, i, p, p,
                                C.c_longlong, i, i, C.POINTER(C.c_float), C.POINTER(C.c_int32),
                                C.POINTER(C.c_float), p],
        "icr_layer_forward": [p, C.POINTER(BatchC), i, p, p, p],
        "icr_seq_logits": [p, C.POINTER(C.c_int32), i, p, p],
        "icr_linear_bf16": [p, p, p, i, i, i, p, p, i, C.POINTER(C.c_int32), p],
        "icr_paged_attention": [p, p, p, i, i, i, i, i, C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int32), i, i, p,
                                C.POINTER(C.c_int32), p],
    }
    for name, argtypes in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = C.c_int
    lib.icr_last_error.restype = C.c_char_p
    lib.icr_last_error.argtypes = []
    lib.icr_abi_version.restype = C.c_int
    lib.icr_num_sms.restype = C.c_int
    _lib = lib
    return lib


def check(status: int) -> None:
    """Map a C status onto the reference's exception classes."""
    if status == 0:
        return
    msg = load().icr_last_error().decode(errors="replace")
    raise _STATUS.get(status, DeviceError)(msg)


def i32_ptr(arr):
    """ctypes int32 pointer to a contiguous numpy int32 array (kept alive by the caller)."""
    return arr.ctypes.data_as(C.POINTER(C.c_int32))


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
