"""ctypes binding of the C ABI in ``include/sfft_b200.h`` (libsfft_b200.so).

There is no CPU fallback: importing a compute entry point without the built
library, or calling one without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libsfft_b200.so"

_i32, _i64, _dbl, _vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p
_int = C.c_int

# name -> (restype, argtypes); pointers are passed as integers (c_void_p)
_SIGS = {
    "sfft_abi_version": (_int, []),
    "sfft_launch_count": (C.c_longlong, []),
    "sfft_profile_enable": (_int, [_int]),
    "sfft_profile_collect": (_int, [_int, _vp, _vp]),
    "sfft_error_string": (C.c_char_p, [_int]),
    "sfft_device_info": (_int, [_vp, _vp, _vp]),
    "sfft_copy_async": (_int, [_vp, _vp, _i64, _vp]),
    "sfft_zero_async": (_int, [_vp, _i64, _vp]),
    "sfft_line_points": (_int, [_vp, _int, _int, _int, _vp, _vp]),
    "sfft_masks_covered": (_int, [_vp, _i64, _vp, _vp]),
    "sfft_alias_scratch_words": (_i64, [_vp, _int]),
    "sfft_alias_masks": (_int, [_vp, _i64, _int, _i64, _vp, _vp, _int, _vp, _i64, _vp, _vp, _vp]),
    "sfft_alias_masks_range": (_int, [_vp, _i64, _int, _i64, _vp, _vp, _int, _int, _vp, _i64, _vp, _vp, _vp]),
    "sfft_lattice_tables": (_int, [_vp, _int, _vp, _vp, _vp]),
    "sfft_fft_size": (_i64, [_i64]),
    "sfft_fft_table_len": (_i64, [_i64]),
    "sfft_fft_tables": (_int, [_i64, _vp, _vp]),
    "sfft_bluestein_bhat": (_int, [_vp, _int, _i64, _vp, _vp, _vp, _vp]),
    "sfft_bluestein": (_int, [_vp, _int, _int, _i64, _vp, _vp, _vp, _vp, _vp, _int, _vp]),
    "sfft_sample_poly_scratch": (_i64, [_vp, _int, _int, _int, _vp, _int]),
    "sfft_sample_poly": (_int, [_vp, _vp, _int, _int, _int, _vp, _vp, _int, _vp, _int,
                                _vp, _vp, _vp, _vp, _vp, _vp, _i64, _int, _vp, _i64, _vp, _int, _vp]),
    "sfft_sample_poly_run": (_int, [_vp, _vp, _int, _int, _int, _vp, _vp, _int, _vp, _int,
                                _vp, _vp, _vp, _vp, _vp, _vp, _i64, _int, _vp, _i64, _vp, _int, _int, _vp]),
    "sfft_sample_poly_prepare": (_int, [_vp, _vp, _int, _int, _int, _vp, _vp, _int, _vp, _int, _vp, _vp, _vp,
                                        _vp, _vp, _i64, _vp, _vp]),
    "sfft_sample_bspline": (_int, [_int, _vp, _vp, _vp, _vp, _int, _int, _vp, _vp, _int, _vp, _int,
                                   _vp, _vp, _i64, _int, _vp, _int, _vp]),
    "sfft_finish_samples": (_int, [_vp, _int, _int, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _int, _vp]),
    "sfft_unit_norm2": (_int, [_vp, _int, _int, _vp, _i64, _vp, _vp, _int, _vp]),
    "sfft_finish_devnoise": (_int, [_vp, _int, _int, _vp, _vp, _i64, _vp, _dbl, _dbl, C.c_uint64, C.c_uint64,
                                    _int, _vp, _int, _vp]),
    "sfft_lattice_nodes": (_int, [_vp, _vp, _int, _int, _int, _int, _vp, _vp, _vp]),
    "sfft_gather_select": (_int, [_vp, _i64, _int, _i64, _vp, _vp, _int, _vp, _vp, _i64, _int, _int,
                                  _dbl, _vp, _vp, _vp, _vp]),
    "sfft_gather_units": (_int, [_vp, _i64, _int, _i64, _vp, _vp, _int, _vp, _vp, _i64, _int, _vp, _int, _vp, _vp]),
    "sfft_combine_units": (_int, [_i64, _int, _vp, _vp, _vp, _int, _int, _int, _dbl, _vp, _vp, _vp, _vp]),
    "sfft_mask_tiles_len": (_i64, [_i64, _int]),
    "sfft_mask_tiles": (_int, [_vp, _i64, _int, _vp, _vp, _i64, _int, _vp, _vp]),
    "sfft_pack_units": (_int, [_vp, _i64, _int, _i64, _vp, _vp, _int, _vp, _vp, _i64, _int, _vp, _int, _vp, _i64,
                               _vp, _vp, _vp]),
    "sfft_combine_slice": (_int, [_i64, _int, _vp, _vp, _i64, _int, _vp, _vp, _int, _dbl, _vp, _vp, _vp, _vp]),
    "sfft_unshard_rows": (_int, [_vp, _int, _int, _int, _i64, _i64, _int, _vp, _vp]),
    "sfft_select_scratch_bytes": (_i64, [_i64]),
    "sfft_select_cap": (_int, [_vp, _vp, _i64, _int, _vp, _vp]),
    "sfft_select_rows_scratch_bytes": (_i64, [_int]),
    "sfft_select_cap_rows": (_int, [_vp, _vp, _i64, _vp, _int, _int, _vp, _vp, _vp]),
    "sfft_scan_scratch_len": (_i64, [_i64]),
    "sfft_flag_indices": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _vp]),
    "sfft_gather_rows": (_int, [_vp, _i64, _int, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "sfft_candidate_product": (_int, [_vp, _i64, _int, _vp, _i64, _vp, _vp]),
    "sfft_residues": (_int, [_vp, _i64, _int, _i64, _vp, _vp, _int, _vp, _vp]),
    "sfft_line_sample_poly": (_int, [_vp, _vp, _int, _int, _int, _int, _vp, _int, _vp, _vp]),
    "sfft_line_sample_poly_all": (_int, [_vp, _vp, _int, _int, _int, _vp, _int, _vp, _vp]),
    "sfft_line_select": (_int, [_vp, _int, _int, _i64, _int, _dbl, _vp, _vp, _vp]),
    "sfft_line_bins": (_int, [_vp, _i64, _int, _int, _i64, _dbl, _vp, _vp, _vp, _vp]),
    "sfft_eval_poly_points": (_int, [_vp, _i64, _int, _vp, _vp, _int, _vp, _vp]),
    "sfft_eval_bspline_points": (_int, [_vp, _i64, _int, _int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sfft_add_noise": (_int, [_vp, _vp, _i64, _dbl, _vp]),
    "sfft_cbc_scan": (_int, [_vp, _vp, _i64, _i64, _i64, _int, _vp, _i64, _vp, _vp]),
    "sfft_prefix_flags": (_int, [_vp, _i64, _int, _vp, _vp]),
    "sfft_scatter_residues": (_int, [_vp, _i64, _int, _i64, _vp, _vp, _vp, _vp]),
    "sfft_pack_rows": (_int, [_vp, _i64, _int, _vp, _vp, _vp]),
    "sfft_cscale": (_int, [_vp, _i64, _dbl, _int, _vp]),
    "sfft_fp64_peak": (_int, [_vp, _int, _int, _vp]),
    "sfft_fp64_mma_peak": (_int, [_vp, _int, _int, _vp]),
    "sfft_l2_random_peak": (_int, [_vp, _i64, _int, _int, _int, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> C.CDLL:
    """Load (building first if the sources are newer) the C-ABI library."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() or os.environ.get("SFFT_B200_REBUILD"):
        try:
            from .build import build
            build()
        except Exception as exc:  # pragma: no cover - depends on toolchain
            raise RuntimeError(
                f"libsfft_b200.so is missing at {LIB_PATH} and could not be built: {exc}"
            ) from exc
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class NativeError(RuntimeError):
    """A CUDA or argument error reported by libsfft_b200 (``code``: its status)."""

    def __init__(self, msg: str, code: int = 0):
        super().__init__(msg)
        self.code = code


E_2BIG = -7  # an argument exceeds a table limit / a scratch is too small


def call(name: str, *args, ctx: str = ""):
    """Invoke an int-returning entry point and raise NativeError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.sfft_error_string(rc).decode()
        where = f" ({ctx})" if ctx else ""
        raise NativeError(f"{name} failed{where}: {msg} [code {rc}]", rc)
    return rc


def query(name: str, *args):
    """Invoke a value-returning entry point (sizes, versions)."""
    return getattr(load(), name)(*args)
