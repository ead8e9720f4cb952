"""ctypes binding of libpsk.so — the C ABI declared in include/psk.h.

The product path has no fallback: if the library is missing or fails to
load, every entry point raises. Errors from the library are raised as
PskError carrying psk_last_error().
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libpsk.so"

PSK_OK = 0
PSK_EINVAL = -1
PSK_ECUDA = -2
PSK_ECAPACITY = -3
PSK_ECAPACITY_NEED = -4
PSK_EUNDERFLOW = -5
PSK_ENOMEM = -6


class PskError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"psk error {code}: {msg}")
        self.code = code


class PoolResult(C.Structure):
    _fields_ = [
        ("status", C.c_int64),
        ("count", C.c_int64),
        ("first_block_id", C.c_int64),
        ("evicted", C.c_int64),
        ("used_blocks", C.c_int64),
        ("matched_tokens", C.c_int64),
        ("lookup_tokens", C.c_int64),
        ("eviction_count", C.c_int64),
        ("next_block_id", C.c_int64),
        ("err_index", C.c_int64),
        ("err_block_id", C.c_int64),
        ("reserved", C.c_int64 * 5),
    ]


class KVLayout(C.Structure):
    _fields_ = [("base", C.c_void_p), ("page_elems", C.c_int64), ("n_layers", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("page_tokens", C.c_int32),
                ("n_pages", C.c_int64)]


class DecodeBatchC(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int32), ("n_sess", C.c_int32), ("n_mod", C.c_int32),
        ("max_rows_per_sess", C.c_int32),
        ("row_mod", C.c_void_p), ("row_sess", C.c_void_p), ("row_in_sess", C.c_void_p),
        ("mod_row_start", C.c_void_p), ("sess_rows", C.c_void_p), ("sess_nrows", C.c_void_p),
        ("sess_len", C.c_void_p), ("sess_pages", C.c_void_p), ("max_sess_pages", C.c_int32),
        ("row_pages", C.c_void_p), ("max_row_pages", C.c_int32),
        ("priv_len", C.c_void_p), ("tokens", C.c_void_p),
    ]


class TinyModelC(C.Structure):
    """psk_tiny_model (include/psk.h)."""
    _fields_ = [("layers", C.c_int32), ("width", C.c_int32), ("heads", C.c_int32), ("context", C.c_int32),
                ("vocab", C.c_int32), ("tok_emb", C.c_void_p), ("prev_emb", C.c_void_p),
                ("pos_emb", C.c_void_p), ("lnf_g", C.c_void_p), ("lnf_b", C.c_void_p), ("head", C.c_void_p),
                ("blocks", C.c_void_p)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_U64 = C.c_uint64
_F = C.c_float

# name -> argtypes (restype is int unless listed in _RESTYPE)
_SIGS: dict[str, list] = {
    "psk_abi_version": [],
    "psk_last_error": [],
    "psk_sm_count": [C.c_int, C.POINTER(_I32)],
    "psk_set_sm_budget": [_I32],
    "psk_get_sm_budget": [C.POINTER(_I32)],
    "psk_init_normal_bf16": [_P, _I64, _U64, _F, _P],
    "psk_fill_bf16": [_P, _I64, _F, _P],
    # K7 pool
    "psk_pool_create": [C.POINTER(_P), _I64, _I32, _I64, _I64, C.c_int],
    "psk_pool_destroy": [_P],
    "psk_pool_reserve": [_P, _I64],
    "psk_pool_records": [_P],
    "psk_pool_host_buffers": [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                              C.POINTER(_P), C.POINTER(_P)],
    "psk_pool_device_out_slots": [_P, C.POINTER(_P)],
    "psk_pool_lookup": [_P, _I32, _P, _I64, _I64, _I32, _P],
    "psk_pool_insert": [_P, _I32, _P, _I64, _I64, _P],
    "psk_pool_evict_until": [_P, _I64, _P],
    "psk_pool_pin": [_P, _I64, _I64, _P],
    "psk_pool_release": [_P, _I64, _P],
    "psk_pool_footprint": [_P, _I32, C.POINTER(_I64), C.POINTER(_I64)],
    "psk_pool_snapshot": [_P, _P, _P, _P, _P, _P, _P, _P],
    "psk_pool_read_record": [_P, _I32, _P, _P],
    # decode step (K5 / K6)
    "psk_embed_rows": [C.POINTER(DecodeBatchC), _P, _I32, _P, _P],
    "psk_rmsnorm_rows": [_P, _I32, _I32, _P, _P, _F, _P, _P],
    "psk_gemv": [_P, _I32, _I32, _P, _P, _I32, _I32, _I32, _I32, _P, _P],
    "psk_gemv_tc": [_P, _I32, _I32, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P],
    "psk_gemv_tc_workspace": [C.POINTER(_I64)],
    "psk_gemv_tc_resid_norm": [_P, _I32, _I32, _P, _P, _I32, _I32, _I32, _P, _P, _P, _F, _P, _P, _P],
    "psk_gemv_tc_qkv_rope": [_P, _I32, _P, C.POINTER(DecodeBatchC), _I32, _I32, _P, _I32, KVLayout, _P, _P, _P],
    "psk_rope_append": [C.POINTER(DecodeBatchC), _P, _I32, _P, _I32, KVLayout, _P, _P],
    "psk_decode_attn_workspace": [C.POINTER(DecodeBatchC), _I32, _I32, C.POINTER(_I64)],
    "psk_decode_attn_kernels": [C.POINTER(DecodeBatchC), _I32, _I32, _I32, C.POINTER(_I32)],
    "psk_decode_attn": [C.POINTER(DecodeBatchC), _P, _I32, _I32, KVLayout, _I32, _P, _P, _P],
    "psk_decode_attn_trace_ring": [_P, _I64, C.POINTER(_I32), C.POINTER(_I32)],
    "psk_gemv_tc_trace_ring": [_P, _I64, _P, C.POINTER(_I32), C.POINTER(_I32)],
    "psk_argmax_advance": [C.POINTER(DecodeBatchC), _P, _I32, _P, _I32, _P],
    "psk_argmax_rows": [_P, _I32, _I32, _P, _P],
    # prefill (K1-K3)
    "psk_gemm": [_P, _P, _I32, _I32, _I32, _I32, _P, _I64, _P],
    "psk_gemm_workspace": [C.POINTER(_I64)],
    "psk_gemm_bind_workspace": [_P, _I64],
    "psk_gemm_qkv_rope_kv": [_P, _P, _I32, _I32, _I32, _P, _I32, KVLayout, _I32, _P, _P, _P],
    "psk_prefill_attn": [_P, _I32, _I32, _I32, KVLayout, _I32, _P, _P, _P],
    "psk_prefill_attn_batch": [_P, _I32, _P, _I32, KVLayout, _I32, _P, _P, _P],
    "psk_gemm_qkv_rope_kv_rows": [_P, _P, _I32, _I32, _I32, _P, _P, _P, KVLayout, _I32, _P, _P],
    "psk_embed_tokens": [_P, _I32, _P, _I32, _P, _P],
    "psk_kv_copy_pages": [_P, _P, _P, _P, _I32, _I64, _P],
    "psk_tiny_scratch_floats": [_P, _I32, _I32, _P],
    "psk_tiny_forward": [_P, _I32, _I32, _I32, _P, _P, _P, _I32, _P, _I64, _P, _P, _P],
}
_RESTYPE = {
    "psk_last_error": C.c_char_p,
    "psk_pool_records": _I64,
}

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load libpsk.so (built in-tree by paper_2602_12029_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("PSK_LIB", str(LIB_PATH)))  # tuning variants (build --define/--out)
    if not path.exists():
        raise PskError(PSK_EINVAL, f"{LIB_PATH} missing: run `python -m paper_2602_12029_b200.build` "
                                   "(the CUDA extension is required; there is no CPU fallback)")
    lib = C.CDLL(str(path), mode=os.RTLD_LOCAL | os.RTLD_NOW)
    for name, args in _SIGS.items():
        if "PSK_LIB" in os.environ and not hasattr(lib, name):
            continue  # an older tuning variant (A/B builds) may lack newer entry points
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    _lib = lib
    return lib


def declared_symbols() -> list[str]:
    return list(_SIGS)


def last_error() -> str:
    msg = load().psk_last_error()
    return msg.decode() if msg else ""


def check(code: int) -> int:
    if code != PSK_OK:
        raise PskError(code, last_error())
    return code


def call(name: str, *args) -> int:
    """Call an int-returning entry point and raise on failure."""
    return check(getattr(load(), name)(*args))


_gemm_ws = None


def bind_gemm_workspace(device) -> None:
    """Allocate (once per process) and bind the prefill GEMMs' split-K
    workspace (psk_gemm_bind_workspace); kept alive for the process."""
    global _gemm_ws
    if _gemm_ws is not None:
        return
    import torch
    nb = C.c_int64()
    check(load().psk_gemm_workspace(C.byref(nb)))
    _gemm_ws = torch.zeros(nb.value, dtype=torch.uint8, device=device)
    check(load().psk_gemm_bind_workspace(_gemm_ws.data_ptr(), nb.value))


def sm_budget() -> int:
    """SMs the persistent kernels currently size their grids for."""
    v = _I32()
    check(load().psk_get_sm_budget(C.byref(v)))
    return int(v.value)


def set_sm_budget(n: int) -> None:
    """0 = all SMs; else the grid budget for the launches (and graph
    captures) that follow, process-wide."""
    check(load().psk_set_sm_budget(int(n)))
