"""ctypes bindings of the in-tree native libraries.

libbs_exec.so is the product path (kernels + executor); it is required and
its absence is an error, never a fallback. libbs_host.so is the CPU-only
scheduler library and libbs_nets.so the CPU-only network definitions
(both usable without a GPU).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"


class BsError(RuntimeError):
    pass


class bs_conv_desc(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "H", "W", "Cin", "Ho", "Wo", "KH", "KW", "stride", "pad", "N",
        "in_ldc", "in_coff", "out_ldc", "out_coff", "res_ldc", "res_coff",
        "relu", "round_out", "split")]


_exec = None
_host = None
_nets = None

FP = C.POINTER(C.c_float)


def _declare_exec(lib: C.CDLL) -> None:
    lib.bs_last_error.restype = C.c_char_p
    lib.bs_kernel_conv.argtypes = [C.POINTER(bs_conv_desc), C.c_int, FP, FP, FP, FP, FP,
                                   C.c_int, FP]
    lib.bs_kernel_conv.restype = C.c_int


def exec_lib() -> C.CDLL:
    """Load libbs_exec.so (raises if it was not built: there is no fallback)."""
    global _exec
    if _exec is None:
        path = LIB_DIR / "libbs_exec.so"
        if not path.exists():
            raise BsError(f"{path} missing: run __graft_entry__.build() (no CPU fallback exists)")
        lib = C.CDLL(str(path))
        _declare_exec(lib)
        _exec = lib
    return _exec


def nets_lib() -> C.CDLL:
    """Load libbs_nets.so: network definitions, weights and images on the
    host (no CUDA; the oracles and bench.py's reference arm use it)."""
    global _nets
    if _nets is None:
        path = LIB_DIR / "libbs_nets.so"
        if not path.exists():
            raise BsError(f"{path} missing: run __graft_entry__.build()")
        lib = C.CDLL(str(path))
        lib.bs_nets_last_error.restype = C.c_char_p
        lib.bs_describe_suite.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        lib.bs_suite_weights_host.argtypes = [C.c_char_p, FP, C.c_size_t]
        lib.bs_make_image.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, FP]
        lib.bs_nets_free.argtypes = [C.c_void_p]
        lib.bs_nets_free.restype = None
        _nets = lib
    return _nets


def nets_check(rc: int) -> None:
    if rc != 0:
        msg = nets_lib().bs_nets_last_error()
        text = msg.decode() if msg else ""
        if rc == -1:
            raise ValueError(text)
        raise BsError(f"status {rc}: {text}")


def host_lib() -> C.CDLL:
    global _host
    if _host is None:
        path = LIB_DIR / "libbs_host.so"
        if not path.exists():
            raise BsError(f"{path} missing: run __graft_entry__.build()")
        _host = C.CDLL(str(path))
    return _host


def check(rc: int, lib: C.CDLL | None = None) -> None:
    if rc != 0:
        lib = lib or exec_lib()
        msg = lib.bs_last_error()
        raise BsError(f"status {rc}: {msg.decode() if msg else ''}")


def fptr(a) -> "C._Pointer":
    """float* of a C-contiguous float32 numpy array (or None)."""
    if a is None:
        return None
    assert a.dtype.name == "float32" and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(FP)


def host_call(job: dict | str) -> str:
    """Run one JSON job through libbs_host.so (bs_host_call); returns JSONL."""
    import json as _json
    lib = host_lib()
    if not getattr(lib, "_bs_declared", False):
        lib.bs_host_call.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        lib.bs_host_call.restype = C.c_int
        lib.bs_host_free.argtypes = [C.c_void_p]
        lib.bs_host_last_error.restype = C.c_char_p
        lib._bs_declared = True
    text = job if isinstance(job, str) else _json.dumps(job)
    out = C.c_void_p()
    rc = lib.bs_host_call(text.encode(), C.byref(out))
    if rc != 0:
        raise BsError(f"bs_host_call status {rc}: {lib.bs_host_last_error().decode()}")
    try:
        return C.string_at(out).decode()
    finally:
        lib.bs_host_free(out)
