"""C-ABI boundary checks that need no GPU: libhx.so loads, exports every symbol
include/hx.h declares, and the ctypes binding types every one of them."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "hx.h"
LIB = ROOT / "paper_2507_00394_b200" / "libhx.so"


def declared() -> list[str]:
    return re.findall(r"^HX_API\s+[\w ]+?\s+(hx_\w+)\(", HEADER.read_text(), flags=re.M)


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        subprocess.run(["make", "-C", str(ROOT), "-j", "8"], check=True, capture_output=True)
    return ctypes.CDLL(str(LIB))


def test_header_declares_the_entry_points():
    names = declared()
    for must in ("hx_gemm", "hx_ln_fwd", "hx_ln_bwd", "hx_attn_fwd", "hx_attn_bwd", "hx_mse_loss",
                 "hx_axpy_f32", "hx_zero", "hx_version", "hx_launch_count"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared():
        assert hasattr(lib, name), name


def test_ctypes_binding_covers_header():
    from paper_2507_00394_b200.runtime import _lib
    assert set(_lib.SIGNATURES) == set(declared())


def test_version_and_counter_callable_without_gpu(lib):
    from paper_2507_00394_b200.runtime import _lib
    L = _lib.load()
    assert L.hx_version() >= 100
    assert L.hx_launch_count() >= 0


def test_argument_checks_fire_before_any_device_work():
    from paper_2507_00394_b200.runtime import _lib
    L = _lib.load()
    # bad shapes are rejected on the host (no CUDA call made)
    assert L.hx_gemm(None, 8, 0, None, 8, 1, None, 8, 0, 8, 8, 0, None, 0, None, 0, None) == 1001
    assert L.hx_attn_fwd(None, 384, None, 128, None, 16, 1, 1, 96, None) == 1003
    assert L.hx_ln_fwd(None, None, None, None, 4, 12, None) == 1001


def test_round2_entry_points_check_arguments_on_the_host():
    from paper_2507_00394_b200.runtime import _lib
    L = _lib.load()
    assert L.hx_attn_bwd_ws_bytes(32768, 1, 16, 128) == 32768 * 16 * 128 * 4
    assert L.hx_attn_bwd_ws_bytes(0, 1, 16, 128) == 0
    assert L.hx_attn_bwd_delta(None, None, 128, None, 16, 1, 1, 96, None) == 1003      # head_dim
    assert L.hx_embed_fwd(None, None, None, None, 16, 1, 12, None) == 1001             # h % 8
    assert L.hx_embed_bwd(None, None, None, None, 0, 1, 64, None) == 1001
    assert L.hx_ce_loss(None, 1024, None, 4, 1000, 992, 1.0, None, None, None) == 1001  # vpad < vocab
