"""CPU checks of the C-ABI boundary: the library builds/loads without a GPU and
exports every symbol include/shiftadd_b200.h declares; the ctypes table
binds exactly that set. No compute calls here."""

import os
import re
import subprocess

import pytest

from paper_2306_06446_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "shiftadd_b200.h")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sa_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2306_06446_b200 import build
        build.build()
    return _lib.load()


def test_header_declares_entry_points():
    syms = header_symbols()
    for must in ("sa_sign_hash", "sa_linear_binary_attn", "sa_hamming_attn", "sa_shift_linear",
                 "sa_quantize_shift", "sa_moe_route", "sa_moe_linear", "sa_moe_mlp", "sa_gemm"):
        assert must in syms


def test_library_exports_every_header_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (sa_[a-z0-9_]+)$", out, flags=re.M))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_ctypes_table_matches_header(lib):
    assert sorted(_lib.symbols()) == header_symbols()
    for name in header_symbols():
        assert getattr(lib, name) is not None


def test_version_and_error_text(lib):
    assert b"sm_100a" in lib.sa_version()
    assert isinstance(lib.sa_last_error(), bytes)


def test_shape_errors_map_without_gpu(lib):
    # argument validation runs on the host before any launch
    with pytest.raises(_lib.ShapeError):
        _lib.call("sa_sign_hash", None, 1, 4, 48, 5, None, None, None, 0, None)
    with pytest.raises(ValueError):
        _lib.call("sa_quantize_shift", None, 4, 3, 3, None, None, None, None)
    with pytest.raises(_lib.ShapeError):
        _lib.call("sa_linear_binary_attn", None, None, None, None, None, None, None,
                  1, 10, 96, 1, 1e-6, None, 0, None)


def test_sm100a_cubin_present(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_library_has_no_debug_state():
    """The product .so carries no sa_debug_* variant switches and no probe
    kernels; those live in the -DSA_DEBUG build only."""
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sa_debug_" not in out and "sa_probe" not in out and "probe_kernel" not in out
    if os.path.exists(_lib.DEBUG_LIB_PATH):
        dbg = subprocess.run(["nm", "-D", "--defined-only", _lib.DEBUG_LIB_PATH],
                             capture_output=True, text=True, check=True).stdout
        assert "sa_debug_attn_mode" in dbg and "sa_probe_mma" in dbg


def test_quant_range_checks_match_device_packing():
    from paper_2306_06446_b200 import quantize as Q
    with pytest.raises(ValueError):
        Q.QuantConfig(p_min=-20, p_max=20)
    with pytest.raises(ValueError):
        Q.QuantConfig(p_min=-130, p_max=-110)
    Q.QuantConfig(p_min=-16, p_max=15)   # 31-wide: fits the 5-bit code
