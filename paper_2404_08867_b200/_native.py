"""ctypes binding of liblq.so (include/lq.h).

The product path has no CPU fallback: if the shared library or a B200 is
missing, every entry point raises ``NativeUnavailable`` loudly.
"""

from __future__ import annotations

import collections
import ctypes as C
import os
import sys
import threading

import numpy as np

from .lower import INSN_DTYPE

__all__ = ["lib", "ctx", "NativeUnavailable", "check", "LQ_TILE", "LQ_SUPER_TILES",
           "LQ_NODE_BLOCK", "Integrand", "Program", "Factor", "LIB_PATH"]

LIB_PATH = os.environ.get("LQ_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblq.so")

LQ_OK, LQ_ERR_VALUE, LQ_ERR_OVERFLOW, LQ_ERR_GRIDCAP = 0, -1, -2, -3
LQ_ERR_CUDA, LQ_ERR_UNSUPPORTED, LQ_ERR_NOMEM = -4, -5, -6
LQ_TILE, LQ_SUPER_TILES, LQ_NODE_BLOCK = 4096, 1024, 256
LQ_FACTOR_SUPPLIED = 1

ABI_VERSION = 11   # LQ_ABI_VERSION of include/lq.h these ctypes structs match
FAM = {"program": 0, "lin_exp": 1, "lin_sincos": 2, "lin_expabs": 3, "quad_exp": 4, "lin_pow": 5, "quad_sincos": 6,
       "prod_quad": 7, "lin_prog": 8}


class NativeUnavailable(RuntimeError):
    """liblq.so could not be loaded or no sm_100 device is usable."""


class Insn(C.Structure):
    _fields_ = [("op", C.c_int32), ("a", C.c_int32), ("b", C.c_int32), ("n", C.c_int32), ("c", C.c_double)]


assert C.sizeof(Insn) == INSN_DTYPE.itemsize


class Program(C.Structure):
    _fields_ = [("insn", C.c_void_p), ("n_insn", C.c_int32), ("n_slots", C.c_int32),
                ("result", C.c_int32), ("n_vars", C.c_int32), ("jit", C.c_void_p)]


class Integrand(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32), ("beta", C.c_void_p), ("gamma", C.c_void_p),
                ("alpha", C.c_double), ("K", C.c_double), ("A", C.c_double), ("B", C.c_double),
                ("C0", C.c_double), ("kappa", C.c_double), ("power", C.c_double), ("prog", Program),
                ("outer", Program)]


class Factor(C.Structure):
    _fields_ = [("count", C.c_int32), ("r_off", C.c_int32), ("r_len", C.c_int32), ("r_result", C.c_int32),
                ("p_off", C.c_int32), ("p_len", C.c_int32), ("p_result", C.c_int32), ("n_slots", C.c_int32),
                ("node_off", C.c_int32), ("reserved", C.c_int32)]


_P = C.c_void_p
_SIGS = {
    "lq_ctx_create": [C.c_int, C.POINTER(C.c_void_p)],
    "lq_ctx_destroy": [_P],
    "lq_ctx_set_stream": [_P, _P],
    "lq_sync": [_P],
    "lq_abi_version": [],
    "lq_device_info": [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "lq_ctx_enable_timing": [_P, C.c_int],
    "lq_last_kernel_ms": [_P, C.POINTER(C.c_float), C.POINTER(C.c_int64)],
    "lq_ctx_transfer_bytes": [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "lq_points_block": [_P, C.c_int32, C.c_uint64, _P, C.c_int64, C.c_int64, _P, C.c_int32],
    "lq_lattice_sum": [_P, C.POINTER(Integrand), C.c_uint64, _P, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)],
    "lq_lattice_partials": [_P, C.POINTER(Integrand), C.c_uint64, _P, C.c_int64, C.c_int64, _P],
    "lq_lattice_layout": [C.POINTER(Integrand), C.c_uint64, _P, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                          C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int64)],
    "lq_reduce_sum": [_P, _P, C.c_int64, C.POINTER(C.c_double)],
    "lq_layout_cover": [C.POINTER(Integrand), C.c_uint64, _P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "lq_mc_sum": [_P, C.POINTER(Program), C.c_int32, C.c_uint64, _P, _P, C.c_uint64, C.c_uint64,
                  C.POINTER(C.c_double)],
    "lq_tensor_sum": [_P, C.POINTER(Program), C.c_int32, _P, _P, C.c_int32, C.c_uint64, C.c_uint64,
                      C.POINTER(C.c_double)],
    "lq_eval_array": [_P, C.POINTER(Program), _P, C.c_int64, C.c_int32, _P],
    "lq_tensor_partials": [_P, C.POINTER(Program), C.c_int32, _P, _P, C.c_int32, C.c_uint64, C.c_int64,
                           C.c_int64, _P],
    "lq_mdi_expabs_partials": [_P, C.c_int32, _P, _P, C.c_double, _P, _P, C.c_int32, C.c_double, C.c_int32,
                               C.c_int32, _P],
    "lq_mdi_block_sums": [_P, _P, C.c_int32, _P, C.c_int32, _P, C.c_int64, C.c_int32, C.c_int32, _P],
    "lq_mdi_combine": [_P, _P, _P, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, C.c_int32, _P],
    "lq_mdi_sum": [_P, _P, C.c_int32, _P, C.c_int32, _P, C.c_int64, _P, _P, _P, _P, _P, C.c_int32, _P],
    "lq_mdi_expabs": [_P, C.c_int32, _P, _P, C.c_double, _P, _P, C.c_int32, C.c_double, _P, _P],
    "lq_mdi_linform2": [_P, C.POINTER(Program), C.c_int32, _P, _P, _P, C.c_double, C.c_int64, C.c_double,
                        C.c_int64, C.c_int32, C.c_int32, _P, C.c_int64, C.POINTER(C.c_double)],
    "lq_mdi_linform_w": [_P, C.POINTER(Program), C.c_int32, _P, _P, _P, C.c_double, C.c_double, C.c_int64,
                         C.c_int32, C.c_int32, _P, C.c_int64, C.POINTER(C.c_double)],
    "lq_mdi_linform": [_P, C.POINTER(Program), C.c_int32, _P, _P, C.c_double, C.c_double, C.c_int64, C.c_int32,
                       C.c_int32, _P, C.c_int64, C.POINTER(C.c_double)],
    "lq_fp64_peak": [_P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_float)],
    "lq_bprod_sum": [_P, C.c_int32, C.c_int32, C.c_uint64, _P, _P, C.c_double, C.c_uint64, C.c_uint64,
                     C.POINTER(C.c_double)],
    "lq_cbc_construct": [_P, C.c_uint64, C.c_int32, _P, C.c_double, _P, C.c_int64, _P],
    "lq_korobov_values": [_P, C.c_uint64, C.c_int32, _P, C.c_double, _P, C.c_int64, _P],
    "lq_jit_create": [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int64],
    "lq_jit_destroy": [_P],
}

_lib = None
_lock = threading.Lock()
_environ = os.environ
_ctxs = {}


def lib():
    """Load liblq.so once (raises NativeUnavailable if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
            h = C.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                fn = getattr(h, name)
                fn.argtypes = args
                fn.restype = C.c_int
            h.lq_last_error.argtypes = []
            h.lq_last_error.restype = C.c_char_p
            got = h.lq_abi_version()
            if got != ABI_VERSION:
                raise NativeUnavailable(f"{LIB_PATH} has ABI {got}, these bindings need {ABI_VERSION}; rebuild it")
            _lib = h
    return _lib


def check(rc):
    if rc == LQ_OK:
        return
    msg = lib().lq_last_error().decode(errors="replace")
    if rc == LQ_ERR_VALUE:
        raise ValueError(msg)
    if rc == LQ_ERR_OVERFLOW:
        raise OverflowError(msg)
    if rc == LQ_ERR_GRIDCAP:
        from .mdi import GridCapError
        raise GridCapError(msg)
    if rc == LQ_ERR_UNSUPPORTED:
        raise NativeUnavailable(msg) if "sm_100a" in msg else NotImplementedError(msg)
    raise RuntimeError(f"liblq error {rc}: {msg}")


class _Ctx:
    def __init__(self, device):
        h = lib()
        p = C.c_void_p()
        rc = h.lq_ctx_create(int(device), C.byref(p))
        if rc != LQ_OK:
            msg = h.lq_last_error().decode(errors="replace")
            raise NativeUnavailable(f"cannot create liblq context on device {device}: {msg}")
        self.ptr = p
        self.device = device

    def __del__(self):
        try:
            if self.ptr:
                lib().lq_ctx_destroy(self.ptr)
        except Exception:
            pass


def _default_device():
    """LQ_DEVICE if set; else torch's current device when the caller has
    initialised CUDA through torch (torchrun scripts set it per rank); else
    LOCAL_RANK, else 0."""
    v = _environ.get("LQ_DEVICE")
    if v is not None:
        return int(v)
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_initialized():
        return torch.cuda.current_device()
    return int(_environ.get("LOCAL_RANK", "0"))


def ctx(device=None):
    """The process's liblq context for ``device`` (default: _default_device)."""
    if device is None:
        device = _default_device()
    key = (device, threading.get_ident())
    c = _ctxs.get(key)
    if c is None:
        c = _ctxs[key] = _Ctx(device)
    return c.ptr


Layout = collections.namedtuple("Layout", "tile_units n_supers n_units mode super_tiles")
LAYOUT_INDEX, LAYOUT_ORBIT, LAYOUT_PAIRED, LAYOUT_ORBIT_FFT, LAYOUT_ORBIT_POW2 = 0, 1, 2, 3, 4


def lattice_layout(pi_struct, n, z=None):
    """Reduction layout liblq uses for the full-lattice sum of (f, n, z):
    units per tile, super-chunks, units, and the mode (LAYOUT_INDEX: units are
    points; LAYOUT_ORBIT: units are chains of mirrored Korobov points;
    LAYOUT_PAIRED: units are mirror-pair indices i in [0, n/2])."""
    tp, ns, nu, mode, st = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32(), C.c_int64()
    check(lib().lq_lattice_layout(C.byref(pi_struct), int(n), as_ptr(z), C.byref(tp), C.byref(ns),
                                  C.byref(nu), C.byref(mode), C.byref(st)))
    return Layout(tp.value, ns.value, nu.value, mode.value, st.value)


def as_ptr(arr):
    # a plain int: the argtypes convert it (a c_void_p wrapper costs ~1 us)
    return arr.ctypes.data if arr is not None else None


def u64(seq):
    return np.ascontiguousarray(np.asarray(seq, dtype=np.uint64))
