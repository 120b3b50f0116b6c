"""ctypes binding of libshiftadd_b200.so (the C-ABI in include/shiftadd_b200.h).

There is no CPU or PyTorch fallback: if the library is missing or cannot be
loaded, every op raises. Status codes map back to the reference's exception
types (ref tensor.py:25-30): SA_ERR_SHAPE → ShapeError, SA_ERR_VALUE →
ValueError, SA_ERR_STATE → StateError, SA_ERR_CUDA → RuntimeError.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libshiftadd_b200.so")
# same sources with -DSA_DEBUG: sa_debug_* kernel-variant setters + MMA probes
DEBUG_LIB_PATH = os.path.join(HERE, "libshiftadd_b200_debug.so")

SA_OK, SA_ERR_SHAPE, SA_ERR_VALUE, SA_ERR_CUDA, SA_ERR_STATE = 0, 1, 2, 3, 4
SA_W_DENSE, SA_W_SHIFT = 0, 1


class ShapeError(ValueError):
    """Operand extents do not line up (ref tensor.py:25-26)."""


class StateError(RuntimeError):
    """Backward / plan requested without the state it needs (ref tensor.py:29-30)."""


_P, _I64, _I32, _F32, _SZ, _U64 = C.c_void_p, C.c_int64, C.c_int, C.c_float, C.c_size_t, C.c_uint64

_SIGS = {
    "sa_version": (C.c_char_p, []),
    "sa_last_error": (C.c_char_p, []),
    "sa_device_info": (_I32, [_P, _P, _P]),
    "sa_launch_count": (_U64, []),
    "sa_sign_hash_workspace": (_SZ, [_I64, _I64, _I64, _I64]),
    "sa_sign_hash": (_I32, [_P, _I64, _I64, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "sa_linear_binary_attn_workspace": (_SZ, [_I64, _I64, _I64, _I64]),
    "sa_linear_binary_attn": (_I32, [_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _F32,
                                     _P, _SZ, _P]),
    "sa_hamming_attn": (_I32, [_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _F32, _P]),
    "sa_binary_popcounts": (_I32, [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
    "sa_dwconv_tokens": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I32, _P]),
    "sa_quantize_shift": (_I32, [_P, _I64, _I32, _I32, _P, _P, _P, _P]),
    "sa_shift_linear": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I32, _I32, _P]),
    "sa_add_linear": (_I32, [_P, _P, C.c_double, _P, _I64, _I64, _I64, _P]),
    "sa_linear": (_I32, [_P, _P, _I32, _P, _I64, _I64, _I64, _I32, _P, _I32, _P]),
    "sa_mlp_workspace": (_SZ, [_I64, _I64]),
    "sa_mlp": (_I32, [_P, _P, _I32, _P, _I32, _P, _I64, _I64, _I64, _I32, _P, _P, _SZ, _P]),
    "sa_moe_route_workspace": (_SZ, [_I64]),
    "sa_moe_route": (_I32, [_P, _P, _I64, _I64, _F32, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "sa_moe_dispatch": (_I32, [_P, _I64, _F32, _P, _P, _P, _P, _P, _SZ, _P]),
    "sa_ln_route_workspace": (_SZ, [_I64, _I32]),
    "sa_ln_route": (_I32, [_P, _P, _P, _P, _I64, _I64, _F32, _I32, _P, _P, _P, _F32, _P, _P, _P,
                           _P, _P, _SZ, _P]),
    "sa_moe_linear": (_I32, [_P, _P, _P, _P, _P, _P, _I32, _P, _P, _I64, _I64, _I64, _P]),
    "sa_moe_mlp_workspace": (_SZ, [_I64, _I64]),
    "sa_moe_mlp": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _I32, _P, _P, _I64, _I64, _I64, _P,
                          _SZ, _P]),
    "sa_gemm": (_I32, [_P, _P, _P, _I64, _I64, _I64, _P]),
    "sa_layernorm": (_I32, [_P, _P, _P, _P, _I64, _I64, _F32, _P]),
    "sa_patch_embed": (_I32, [_P, _I64, _I64, _I64, _I64, _I64, _F32, _P, _I64, _P, _P, _P, _P]),
    "sa_softmax_attn_strided": (_I32, [_P, _P, _P, _I64, _P, _I64, _I64, _I64, _I64, _P]),
    "sa_softmax_attn": (_I32, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _P]),
    "sa_pool": (_I32, [_P, _P, _I64, _I64, _I64, _I32, _P]),
    "sa_tc_tile_n": (_I32, [_I64]),
    "sa_weight_pack_bytes": (_SZ, [_I64, _I64, _I32, _I32]),
    "sa_weight_pack": (_I32, [_P, _I32, _I64, _I64, _I32, _I32, _P, _P]),
    "sa_tc_linear": (_I32, [_P, _P, _I32, _I32, _P, _I64, _I64, _I64, _P, _I32, _P]),
    "sa_tc_moe_linear_grouped": (_I32, [_P, _P, _P, _P, _P, _P, _I32, _I32, _P, _I64, _I64, _I64,
                                        _P]),
    "sa_tc_moe_linear": (_I32, [_P, _P, _P, _P, _P, _P, _I32, _P, _P, _I64, _I64, _I64, _P]),
    "sa_tc_mlp_workspace": (_SZ, [_I64, _I64]),
    "sa_tc_mlp": (_I32, [_P, _P, _I32, _I32, _P, _I32, _I32, _P, _I64, _I64, _I64, _P, _P, _SZ,
                         _P]),
    "sa_tc_moe_mlp": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _P, _P, _I64, _I64, _I64,
                             _P, _SZ, _P]),
    "sa_tc_patch_embed": (_I32, [_P, _I64, _I64, _I64, _I64, _I64, _F32, _P, _I32, _I64, _P, _P,
                                 _P, _P]),
    "sa_tc_patch_embed_ln_ok": (_I32, [_I64, _I32, _I32]),
    "sa_tc_patch_embed_ln": (_I32, [_P, _I64, _I64, _I64, _I64, _I64, _F32, _P, _I32, _I64, _P,
                                    _P, _F32, _P, _P]),
    "sa_tc_fused_mlp_ok": (_I32, [_I64, _I64]),
    "sa_tc_fused_mlp_w1_bn": (_I32, []),
    "sa_tc_fused_mlp_chunk": (_I32, [_I64]),
    "sa_tc_moe_mlp_fused": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64,
                                   _P]),
    "sa_tc_moe_mlp_fused_ln": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64,
                                      _P, _P, _F32, _P]),
    "sa_tc_mlp_fused": (_I32, [_P, _P, _I32, _P, _I32, _P, _I64, _I64, _I64, _P, _P]),
    "sa_moe_partition_workspace": (_SZ, [_I64]),
    "sa_moe_partition": (_I32, [_P, _I64, _P, _P, _P, _SZ, _P]),
    "sa_ln_qkv_hash_ok": (_I32, [_I64, _I64]),
    "sa_fused_moe_linear_ok": (_I32, [_I64]),
    "sa_fused_moe_linear": (_I32, [_P, _P, _P, _P, _P, _F32, _I64, _I64, _P, _P, _P, _P]),
    "sa_fused_moe_linear_ln_route": (_I32, [_P, _P, _P, _P, _P, _F32, _I64, _I64, _P, _P, _P, _P,
                                            _P, _F32, _P, _P, _P, _P, _P]),
    "sa_ln_qkv_hash_workspace": (_SZ, [_I64, _I64, _I64]),
    "sa_ln_qkv_hash": (_I32, [_P, _P, _P, _F32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _F32, _I64,
                              _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
}

_lib = None
_debug_lib = None
_lock = threading.Lock()


def _open(path):
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2306_06446_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def load():
    """Load (once) and return the ctypes library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            _lib = _open(LIB_PATH)
    return _lib


@contextlib.contextmanager
def debug_library():
    """Route every C-ABI call made inside the block to the debug build (same
    kernels, plus the sa_debug_* variant switches); yields that library.
    Test / diagnostics use only — the product never enters this."""
    global _lib, _debug_lib
    prev = load()
    with _lock:
        if _debug_lib is None:
            _debug_lib = _open(DEBUG_LIB_PATH)
        _lib = _debug_lib
    try:
        yield _debug_lib
    finally:
        _lib = prev


def symbols():
    return sorted(_SIGS)


def last_error() -> str:
    return load().sa_last_error().decode(errors="replace")


def check(status: int, what: str = ""):
    if status == SA_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if status == SA_ERR_SHAPE:
        raise ShapeError(msg)
    if status == SA_ERR_VALUE:
        raise ValueError(msg)
    if status == SA_ERR_STATE:
        raise StateError(msg)
    raise RuntimeError(msg)


def call(name: str, *args):
    """Invoke a C-ABI entry point that returns a status code; raise on error."""
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a contiguous CUDA tensor (None passes NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    return int(load().sa_launch_count())


class Workspace:
    """Grow-only scratch buffer per device (the library never allocates)."""

    _bufs: dict = {}
    # Buffers replaced by a larger one are kept alive, never returned to the
    # caching allocator: a CUDA graph captured while they were current keeps
    # writing to them on every replay (runtime.GraphedForward).
    _retired: list = []

    @classmethod
    def get(cls, nbytes: int, device=None, slot: int = 0) -> torch.Tensor:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        key = (dev.index, slot)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                cls._retired.append(buf)
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
            cls._bufs[key] = buf
        return buf

    @classmethod
    def live(cls) -> list:
        """Every workspace buffer currently allocated (current and retired)."""
        return list(cls._bufs.values()) + list(cls._retired)
