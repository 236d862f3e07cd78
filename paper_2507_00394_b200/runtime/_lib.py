"""ctypes binding of libhx.so (the C-ABI declared in include/hx.h).

There is no fallback: if the shared library is missing or a CUDA device is not
available, every entry point raises :class:`KernelLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent.parent
LIB_PATH = Path(os.environ.get("HX_LIB", _PKG / "libhx.so"))

HX_E = {1001: "HX_E_SHAPE", 1002: "HX_E_ALIGN", 1003: "HX_E_UNSUPPORTED"}

EPI_STORE_BF16, EPI_RESID_BF16, EPI_GELU, EPI_DGELU, EPI_ACC_F32, EPI_STORE_F32 = range(6)

_P = ctypes.c_void_p
_I = ctypes.c_int
_LL = ctypes.c_longlong

# name -> argtypes (restype is int unless listed in _RESTYPE)
SIGNATURES: dict[str, list] = {
    "hx_version": [],
    "hx_launch_count": [],
    "hx_set_sm_reserve": [_I],
    "hx_gemm": [_P, _I, _I, _P, _I, _I, _P, _I, _I, _I, _I, _I, _P, _I, _P, _I, _P],
    "hx_ln_fwd": [_P, _P, _P, _P, _I, _I, _P],
    "hx_ln_bwd": [_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P],
    "hx_attn_fwd": [_P, _I, _P, _I, _P, _I, _I, _I, _I, _P],
    "hx_attn_bwd": [_P, _I, _P, _P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P],
    "hx_attn_bwd_delta": [_P, _P, _I, _P, _I, _I, _I, _I, _P],
    "hx_attn_bwd_ws_bytes": [_I, _I, _I, _I],
    "hx_embed_fwd": [_P, _P, _P, _P, _I, _I, _I, _P],
    "hx_embed_bwd": [_P, _P, _P, _P, _I, _I, _I, _P],
    "hx_ce_loss": [_P, _I, _P, _I, _I, _I, ctypes.c_float, _P, _P, _P],
    "hx_mse_loss": [_P, _LL, _P, _P, _P],
    "hx_axpy_f32": [_P, _P, _LL, _P],
    "hx_zero": [_P, _LL, _P],
}
_RESTYPE = {"hx_launch_count": ctypes.c_longlong, "hx_attn_bwd_ws_bytes": ctypes.c_longlong}


class KernelLibraryError(RuntimeError):
    """libhx could not be loaded or a kernel call failed."""


_lib = None


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the library.  Loading needs no GPU."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise KernelLibraryError(
            f"{p} not found: build it with `make` (or __graft_entry__.build()); "
            "there is no CPU fallback for the stage-execution kernels")
    lib = ctypes.CDLL(str(p))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, ctypes.c_int)
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        label = HX_E.get(rc, f"cudaError {rc}")
        raise KernelLibraryError(f"{what} failed: {label}")


# Optional per-entry-point device timing (bench.py's in-step roofline): while
# enabled, every call is bracketed by CUDA events on the current stream, which
# is the stream every wrapper in kernels.py launches on.
_timers: dict[str, list] | None = None


def start_kernel_timers() -> None:
    global _timers
    _timers = {}


_tagged: dict[str, list] | None = None


def stop_kernel_timers(with_tags: bool = False):
    """Synchronise and return {entry point: {"launches", "total_ms", "mean_ms"}}
    (and, ``with_tags``, the same per call tag, e.g. per GEMM shape)."""
    global _timers, _tagged
    import torch

    timers, _timers = _timers or {}, None
    tagged, _tagged = _tagged or {}, None
    torch.cuda.synchronize()

    def summarise(d):
        out = {}
        for name, evs in d.items():
            tot = sum(a.elapsed_time(b) for a, b in evs)
            out[name] = {"launches": len(evs), "total_ms": tot, "mean_ms": tot / len(evs)}
        return out

    return (summarise(timers), summarise(tagged)) if with_tags else summarise(timers)


def call(name: str, *args, tag: str | None = None) -> None:
    """Invoke a C-ABI entry point; raise on a nonzero return.  While timers run,
    the call is bracketed by CUDA events, keyed by name (and name:tag)."""
    global _tagged
    fn = getattr(load(), name)
    if _timers is None:
        check(fn(*args), name)
        return
    import torch

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rc = fn(*args)
    b.record()
    _timers.setdefault(name, []).append((a, b))
    if tag is not None:
        if _tagged is None:
            _tagged = {}
        _tagged.setdefault(f"{name}:{tag}", []).append((a, b))
    check(rc, name)


def set_sm_reserve(sms: int) -> None:
    """SMs kept free of persistent-kernel CTAs (for NCCL kernels beside them)."""
    check(load().hx_set_sm_reserve(int(sms)), "hx_set_sm_reserve")


def launch_count() -> int:
    return int(load().hx_launch_count())
