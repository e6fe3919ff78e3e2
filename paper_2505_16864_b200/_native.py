"""ctypes binding of the C ABI in ``include/tokencarve_b200.h`` (``_lib/libtcb200.so``).

The library is loaded lazily on first use and the product path fails loudly
(``NativeUnavailable``) when it is missing -- there is no CPU fallback.  Status
codes are mapped back to the reference exception taxonomy (errors.py:4-29).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ContractError, DomainError, ShapeError, SizeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libtcb200.so")

F32, BF16, F16, F64 = 0, 1, 2, 3

_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_U64 = C.c_uint64
_D = C.c_double
_F = C.c_float

# name -> argtypes, mirroring include/tokencarve_b200.h
SIGNATURES = {
    "tcb_last_error": [],
    "tcb_abi_version": [],
    "tcb_curve_build": [_I, _I, _I, _P, _P, _P],
    "tcb_gather_rows": [_P, _P, _P, _I64, _I64, _I64, _P],
    "tcb_adjacency_build": [_P, _I, _I, _I, _I, _I, _I, _P, _P],
    "tcb_block_pool": [_P, _P, _I, _I64, _I64, _I, _I, _I, _I, _I, _I64, _I64, _P, _P, _P],
    "tcb_block_relevance": [_P, _I, _P, _I, _I, _I, _I, _P, _P],
    "tcb_block_select": [_P, _I, _I, _I, _P, _I, _I, _D, _I, _P, _P, _P],
    "tcb_block_scores": [_P, _I, _P, _I, _I, _I, _I, _P, _P],
    "tcb_block_select_scores": [_P, _I, _I, _I, _P, _I, _I, _D, _I, _P, _P, _P],
    "tcb_block_mask": [_P, _I, _P, _I, _I, _I, _I, _P, _I, _I, _D, _P, _P, _P, _I64, _P],
    "tcb_block_mask_scratch": [_I, _I, _I],
    "tcb_mask_pack": [_P, _I64, _I, _I, _P, _P, _P],
    "tcb_mask_unpack": [_P, _I64, _I, _I, _P, _P],
    "tcb_carve_workspace_bytes": [_I, _I, _I, _I, _I],
    "tcb_carve_fwd": [_P, _P, _P, _P, _I, _I64, _I64, _P, _I, _P, _I, _I, _I, _I, _I, _I64,
                      _I64, _F, _P, _I64, _P],
    "tcb_carve_fwd_simt": [_P, _P, _P, _P, _I, _I64, _I64, _P, _I, _P, _I, _I, _I, _I, _I, _I64,
                           _I64, _F, _P],
    "tcb_carve_f32_workspace_bytes": [_I, _I, _I, _I],
    "tcb_carve_fwd_f32": [_P, _P, _P, _P, _I64, _I64, _P, _I, _P, _I, _I, _I, _I, _I, _I64, _I64,
                          _F, _P, _I64, _P, _P],
    "tcb_upsample_renoise": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _D, _I, _U64, _U64, _P],
    "tcb_euler_step": [_P, _P, _P, _I64, _F, _P],
    "tcb_euler_step_f64": [_P, _P, _P, _I64, _D, _P],
    "tcb_upsample_renoise_f64": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _D, _I, _U64, _U64, _P],
    "tcb_upsample_renoise_curve": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _D, _I, _U64,
                                   _U64, _P],
    "tcb_curve_positions": [_P, _I64, _I, _I, _I, _P, _P],
    "tcb_patchify_permute": [_P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P],
    "tcb_unpermute_euler": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _F, _P, _P],
    "tcb_mask_words_to_packbits": [_P, _I64, _I, _I, _P, _P],
    "tcb_packbits_to_dense": [_P, _I64, _I, _P, _P],
    "tcb_rope_permute": [_P, _I64, _I64, _P, _I64, _I64, _P, _I, _P, _I, _I, _I, _I, _I, _P, _I,
                         _I, _I, _P],
}


_I64_RESULT = ("tcb_block_mask_scratch", "tcb_carve_f32_workspace_bytes", "tcb_carve_workspace_bytes")


class NativeUnavailable(RuntimeError):
    """The sm_100a library is not built or cannot be loaded."""


_lock = threading.Lock()
_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing; run `python -m paper_2505_16864_b200._build` "
                "(no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = (C.c_char_p if name == "tcb_last_error" else
                          C.c_int64 if name in _I64_RESULT else C.c_int)
        _lib = lib
    return _lib


_EXC = {1: ShapeError, 2: DomainError, 3: SizeError, 4: ContractError}


def query(name: str, *args) -> int:
    """A C-ABI entry that returns a value instead of a status (no error mapping)."""
    return int(getattr(load(), name)(*args))


def call(name: str, *args) -> None:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.tcb_last_error().decode(errors="replace")
        raise _EXC.get(rc, RuntimeError)(f"{name}: {msg}")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_of(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream
