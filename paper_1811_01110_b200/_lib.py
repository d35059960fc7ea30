"""ctypes binding of the in-tree C-ABI library ``_lib/libgigaqbx_tsqbx.so``.

The library is the product: there is no CPU or eager fallback.  ``load()``
raises if the shared object is missing (run ``__graft_entry__.build()`` or
``make -C paper_1811_01110_b200/csrc``), and every compute entry point raises
if no CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GIGAQBX_LIB_PATH") or os.path.join(HERE, "_lib",
                                                               "libgigaqbx_tsqbx.so")
CSRC = os.path.join(HERE, "csrc")

ABI_VERSION = 12      # TSQBX_ABI_VERSION in include/tsqbx.h

# status codes (include/tsqbx.h)
OK = 0
ERR_SEPARATION = 1
ERR_COINCIDENT = 2
ERR_ARGUMENT = 3
ERR_CUDA = 4

EQ_LAPLACE = 0
EQ_HELMHOLTZ = 1
FLAG_VALIDATE = 1
FLAG_GENERIC = 2
FLAG_REAL_WEIGHTS = 4
FLAG_ONE_TARGET = 8
FLAG_PRECISE = 16
FLAG_UNIFORM_TARGETS = 32
FLAG_KR_NARROW = 64
FLAG_KR_WIDE = 128
FLAG_LONG_ROWS = 1 << 16
FLAG_FLAT = 1 << 17
FLAG_TWO_ROWS = 1 << 18
FLAG_WINDOW = 1 << 19
WINDOW = 128
MAX_ORDER = 64
ERR_KEY_NONE = (1 << 63) - 1
ERR_KEY_SUSPECT = (1 << 63) - 2

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double
_U = ctypes.c_uint

# every symbol declared in include/tsqbx.h with its (restype, argtypes)
SIGNATURES = {
    "tsqbx_abi_version": (_I, []),
    "tsqbx_last_error": (ctypes.c_char_p, []),
    "tsqbx_device_info": (_I, [_P, _P, _P]),
    "tsqbx_packed_doubles": (_I64, [_I64, _I]),
    "tsqbx_pack_sources": (_I, [_I64, _P, _P, _P, _P, _P, _P]),
    "tsqbx_eval_workspace_bytes": (_I64, [_I, _I, _I, _I64]),
    "tsqbx_eval_packed": (_I, [_I, _I, _D, _I, _P, _I64, _I, _P, _I64, _P, _P, _P, _P, _P, _P,
                               _P, _I64, _P, _I64, _I64, _U, _I, _P, _I64, _P, _P, _P]),
    "tsqbx_user_workspace_bytes": (_I64, [_I, _I, _I, _I64, _I64]),
    "tsqbx_eval_laplace": (_I, [_I, _I, _P, _P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _I64, _U,
                                _P, _I64, _P, _P, _P]),
    "tsqbx_eval_helmholtz": (_I, [_I, _D, _I, _P, _P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P,
                                  _I64, _U, _P, _I64, _P, _P, _P]),
    "tsqbx_validate": (_I, [_P, _I64, _P, _I64, _P, _P, _P, _P, _I64, _P, _P]),
    "tsqbx_order_workspace_bytes": (_I64, [_I64]),
    "tsqbx_order_targets": (_I, [_I64, _P, _P, _P, _P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P,
                                 _P, _P]),
    "tsqbx_scatter_c128": (_I, [_I64, _P, _P, _P, _P]),
    "tsqbx_sell_to_csr": (_I, [_I64, _P, _P, _P, _P, _P]),
    "tsqbx_sell_compact": (_I, [_I64, _P, _P, _P, _P, _P]),
    "tsqbx_sell_workspace_bytes": (_I64, [_I64]),
    "tsqbx_sell_size": (_I, [_I64, _P, _P, _I64, _P, _P, _P]),
    "tsqbx_sell_fill": (_I, [_I64, _P, _P, _P, _P, _P]),
    "tsqbx_near_workspace_bytes": (_I64, [_I64, _I64]),
    "tsqbx_near_count": (_I, [_P, _P, _I64, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _P]),
    "tsqbx_near_fill": (_I, [_P, _P, _I64, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "tsqbx_eval_packed_win": (_I, [_I, _I, _D, _I, _P, _I64, _I, _P, _I64, _P, _P, _P, _P, _P, _P,
                                   _P, _P, _P, _I64, _P, _I64, _I64, _U, _I, _P, _I64, _P, _P,
                                   _P]),
    "tsqbx_sell_window": (_I, [_I64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "tsqbx_near_index": (_I, [_P, _P, _I64, _P, _I64, _P, _I64, _P, _P, _P]),
    "tsqbx_fused_scratch_bytes": (_I64, [_I, _I, _I, _I, _I]),
    "tsqbx_eval_fused": (_I, [_I, _D, _I, _P, _I64, _P, _P, _P, _P, _I64, _P, _I64, _P, _I64, _P,
                              _U, _I, _P, _I64, _P, _P, _P]),
    "tsqbx_near_recount": (_I, [_P, _P, _I64, _I64, _P, _I64, _P, _P, _P, _P]),
    "tsqbx_near_mask_bytes": (_I64, [_I64, _I64]),
    "tsqbx_near_recount_masks": (_I, [_P, _P, _I64, _I64, _P, _I64, _P, _P, _P, _P, _I64, _P]),
    "tsqbx_near_fill_masks": (_I, [_P, _P, _I64, _I64, _P, _I64, _P, _P, _P, _P, _P, _P, _I64,
                                   _P]),
    "tsqbx_near_fill_rows": (_I, [_P, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _I64, _P, _P, _P,
                                  _P, _P]),
    "tsqbx_fp64_probe": (_I, [_P, _I64, _I, _I, _P]),
    "tsqbx_one_staging_doubles": (_I64, [_I64, _I]),
    "tsqbx_eval_one": (_I, [_I, _I, _D, _I, _P, _I64, _U, _P, _I64, _P, _P]),
    "tsqbx_box_rows_workspace_bytes": (_I64, [_I64]),
    "tsqbx_box_rows_count": (_I, [_I64, _P, _P, _P, _P, _P, _I64, _P, _I64, _P, _P, _P]),
    "tsqbx_box_rows_fill": (_I, [_I64, _P, _P, _P, _P, _P, _I64, _P, _P, _P]),
    "tsqbx_p2p_workspace_bytes": (_I64, [_I64, _I64, _I64, _I]),
    "tsqbx_p2p_packed": (_I, [_I, _I, _D, _P, _I64, _I, _I64, _P, _P, _P, _P, _P, _I64, _U, _P,
                              _I64, _P, _P, _P]),
    "tsqbx_p2p_find_singular": (_I, [_P, _I64, _I64, _P, _P, _P, _P, _I64, _P, _P]),
    "tsqbx_p2p_user_workspace_bytes": (_I64, [_I, _I64, _I64]),
    "tsqbx_p2p_laplace": (_I, [_I, _P, _P, _P, _I64, _P, _P, _I64, _U, _P, _I64, _P, _P, _P]),
    "tsqbx_p2p_helmholtz": (_I, [_I, _D, _P, _P, _P, _I64, _P, _P, _I64, _U, _P, _I64, _P, _P,
                                 _P]),
}

_lib = None
_lock = threading.Lock()


def build(verbose: bool = False) -> str:
    """Compile the CUDA library in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    jobs = str(max(1, min(8, os.cpu_count() or 1)))
    res = subprocess.run(["make", "-C", CSRC, "-j", jobs], capture_output=not verbose, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"CUDA library build failed:\n{res.stdout}\n{res.stderr}")
    return LIB_PATH


def load():
    """Load the library (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the TSQBX CUDA library must be built "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.tsqbx_abi_version() != ABI_VERSION:
            raise RuntimeError(f"TSQBX ABI version mismatch: library "
                               f"{L.tsqbx_abi_version()}, bindings {ABI_VERSION}")
        _lib = L
    return _lib


def last_error() -> str:
    return load().tsqbx_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != OK:
        raise RuntimeError(f"{what} failed (status {rc}): {last_error()}")
