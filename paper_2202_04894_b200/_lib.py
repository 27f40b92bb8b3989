"""ctypes binding of libdefmm_b200.so (the C-ABI of include/defmm_b200.h).

There is deliberately no fallback: if the library is missing the import of
the compute entry points raises, so a GPU test can never pass on a silent CPU
or eager-PyTorch path.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdefmm_b200.so")

_i32, _i64, _f64, _vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p

# name -> argtypes (all pointers passed as integers / c_void_p)
_SIGS = {
    "defmm_abi_version": [],
    "defmm_last_error": [],
    "defmm_tree_build": [_vp, _i64, _vp, _f64, _i32, _i32, _vp],
    "defmm_tree_ncells": [_vp],
    "defmm_tree_fetch": [_vp] + [_vp] * 7,
    "defmm_tree_free": [_vp],
    "defmm_dtt_build": [_vp, _i32] + [_vp] * 4 + [_vp, _i32] + [_vp] * 4 + [_i32] + [_vp] * 5,
    "defmm_dtt_sizes": [_vp, _vp],
    "defmm_dtt_fetch": [_vp] * 17,
    "defmm_dtt_translations": [_vp, _vp],
    "defmm_dtt_source_hats": [_vp] * 6 + [_i64, _vp, _vp, _vp],
    "defmm_dtt_free": [_vp],
    "defmm_stage_pack": [_i64, _vp, _vp, _vp, _i64, _i32, _vp],
    "defmm_tree_keys": [_i64, _vp, _vp, _f64, _i32, _vp, _vp],
    "defmm_dtt_classify": [_i64] + [_vp] * 6 + [_i64, _i32, _i64] + [_vp] * 7,
    "defmm_fma_peak": [_i32, _i64, _vp, _vp],
    "defmm_l2_stream": [_vp, _i64, _i32, _i32, _vp, _vp],
    "defmm_m2l_canon_c128": [_i32, _i64] + [_vp] * 9,
    "defmm_direct_workspace_bytes": [_i64],
    "defmm_spectrum_stride": [_i32, _i32],
    "defmm_spectral_layout": [_i32, _vp, _vp, _vp],
    "defmm_direct_c128": [_i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _f64, _f64, _vp, _vp, _vp],
}
for _t in ("c128", "c64"):
    _SIGS.update({
        f"defmm_p2m_{_t}": [_i32, _i64] + [_vp] * 12 + [_vp, _f64, _vp, _vp],
        f"defmm_m2m_{_t}": [_i32, _i64, _vp, _vp, _vp, _f64, _vp, _f64, _vp, _vp],
        f"defmm_m2f_{_t}": [_i32, _i64, _vp, _vp, _vp, _vp],
        f"defmm_symbols_{_t}": [_i32, _i64, _vp, _vp, _f64, _vp, _vp],
        f"defmm_expand_symbols_{_t}": [_i32, _i64, _vp, _vp, _vp, _vp, _vp],
        f"defmm_m2l_rows_{_t}": [_i32, _i64] + [_vp] * 7,
        f"defmm_m2l_blocked_{_t}": [_i32, _i64] + [_vp] * 10,
        f"defmm_m2l_group_{_t}": [_i32, _i32, _i64] + [_vp] * 7,
        f"defmm_m2l_stage_{_t}": [_i32, _i64, _i32, _i32] + [_vp] * 11,
        f"defmm_f2l_rows_{_t}": [_i32, _i64, _vp, _vp, _vp, _vp],
        f"defmm_l2l_{_t}": [_i32, _i64, _vp, _vp, _vp, _vp, _vp, _f64, _vp, _f64, _vp, _vp],
        f"defmm_l2p_{_t}": [_i32, _i64] + [_vp] * 13 + [_f64, _vp, _vp, _vp, _vp, _vp],
        f"defmm_p2p_mutual_{_t}": [_i64] + [_vp] * 14 + [_f64, _f64, _vp, _i32, _i32, _vp],
        f"defmm_p2p_gather_{_t}": [_i64] + [_vp] * 11,
        f"defmm_p2p_{_t}": [_i64] + [_vp] * 16 + [_f64, _f64, _vp, _vp, _i64, _vp, _vp, _vp, _i32, _i32, _vp],
    })

EXPORTED = tuple(_SIGS)

_lib = None


class DefmmLibraryError(RuntimeError):
    pass


def load():
    """Load the in-tree library (raises DefmmLibraryError when absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DefmmLibraryError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2202_04894_b200.build` "
            "(there is no CPU fallback for the defmm operators)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _i32
    lib.defmm_tree_ncells.restype = _i64
    lib.defmm_direct_workspace_bytes.restype = _i64
    lib.defmm_tree_free.restype = None
    lib.defmm_dtt_free.restype = None
    lib.defmm_last_error.restype = C.c_char_p
    _lib = lib
    return lib


def check(rc: int, what: str):
    if rc != 0:
        msg = load().defmm_last_error().decode(errors="replace")
        raise DefmmLibraryError(f"{what} failed with status {rc}: {msg}")


def call(name: str, *args):
    """Invoke an operator; tensors are passed by data_ptr()."""
    fn = getattr(load(), name)
    conv = []
    for a in args:
        if hasattr(a, "data_ptr"):
            conv.append(a.data_ptr() if a.numel() else None)
        else:
            conv.append(a)
    check(fn(*conv), name)
