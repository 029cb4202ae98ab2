"""ctypes binding of libkle_b200.so (the C ABI in include/kle_b200.h).

There is no CPU fallback: importing the solver modules without the built
library, or calling them without a CUDA device, raises ``DeviceError``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .core import DeviceError

_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libkle_b200.so"
_lib = None

_p = C.c_void_p
_i = C.c_int
_d = C.c_double
_z = C.c_size_t

_SIGS = {
    "kle_abi_version": ([], _i),
    "kle_last_error": ([], C.c_char_p),
    "kle_release_resources": ([], _i),
    "kle_fine_layout": ([_i, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)], _i),
    "kle_kl_tridiag_f64": ([_p, _i, _i, _p, _i, _d, _p, _p, _p], _i),
    "kle_fine_factor_f64": ([_p, _p, _i, _i, _d, _d, _p, _p], _i),
    "kle_sweep_f64": ([_p, _p, _p, _i, _i, _i, _i, _i, _d, _d, _p], _i),
    "kle_fgr_f64": ([_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _d, _d, _d, _d, _p], _i),
    "kle_cgc_scratch_bytes": ([_i, _i, _i], _z),
    "kle_shift_factor_bytes": ([_i, _i, _i], _z),
    "kle_shift_factor_f64": ([_p, _p, _p, _i, _i, _i, _d, _p, _p], _i),
    "kle_three_step_f64": ([_p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _d, _p, _p, _p, _z, _p], _i),
    "kle_cgc_update_f64": ([_p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _d, _i, _i, _d, _p, _p, _p, _p, _p, _p, _z,
                            _p], _i),
    "kle_pcgc_workspace_bytes": ([_i, _i, _i], _z),
    "kle_imag_residue_scratch_bytes": ([_i, _i, _i], _z),
    "kle_imag_residue_f64": ([_p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _d, _p, _p, _z, _p], _i),
    "kle_pcgc_solve_f64": ([_p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _d, _d, _d, _d, _i, _p, _p, _p, _p,
                            _p, _z, _p], _i),
    "kle_pcgc_solve_ref_f64": ([_p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _d, _d, _d, _d, _i, _p, _i, _p,
                                _p, _p, _p, _p, _p, _p, _z, _p], _i),
    "kle_err_aggregate_f64": ([_p, _p, _i, _i, _i, _i, _p, _p, _p, _p], _i),
    "kle_err_ref_f64": ([_p, _p, _i, _i, _i, _i, _i, _d, _i, _p, _p, _p, _p, _p, _p], _i),
    "kle_parareal_init_f64": ([_p, _p, _p, _i, _i, _i, _d, _d, _p, _p], _i),
    "kle_parareal_step_f64": ([_p, _p, _p, _p, _p, _i, _i, _i, _d, _d, _i, _i, _d, _p, _p, _p, _p, _p], _i),
    "kle_parareal_workspace_bytes": ([_i, _i, _i], _z),
    "kle_parareal_solve_f64": ([_p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _d, _d, _d, _i, _p, _i, _p, _p, _p, _p,
                                _p, _p, _z, _p], _i),
    "kle_newton_work_bytes": ([_i, _i, _i], _z),
    "kle_newton_sweep_f64": ([_i, _p, _p, _p, _i, _i, _i, _i, _i, _d, _d, _d, _d, _d, _i, _p, _p, _p, _z, _p], _i),
    "kle_para_combine_f64": ([_p, _p, _p, _p, _p, _i, _i, _i, _i, _p], _i),
    "kle_newton_cgc_f64": ([_i, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _d, _d, _d, _d, _d, _p, _p, _p], _i),
    "kle_block_dft_f64": ([_p, _p, _i, _i, _i, _p], _i),
    "kle_shifted_tridiag_solve_f64": ([_p, _p, _p, _d, _d, _d, _p, _p, _p, _i, _i, _p, _p], _i),
    "kle_2d_kl5pt_f64": ([_p, _i, _i, _p, _i, _d, _p, _p, _p, _p], _i),
    "kle_2d_factor_f64": ([_p, _p, _p, _i, _i, _p, _i, _d, _d, _p, _p, _p], _i),
    "kle_2d_fine_work_doubles": ([_i, _i, _i], _z),
    "kle_2d_fgr_f64": ([_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _d, _d, _d, _d, _p, _z, _p, _p], _i),
    "kle_2d_sweep_f64": ([_p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _i, _d, _d, _p, _z, _p, _p], _i),
    "kle_2d_fine_stage_doubles": ([_i, _i], _z),
    "kle_2d_fine_stage_f64": ([_p, _p, _i, _i, _p, _p], _i),
    "kle_2d_fgr_staged_f64": ([_p, _p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _d, _d, _d, _d, _p, _z, _p, _p], _i),
    "kle_2d_sweep_staged_f64": ([_p, _p, _i, _i, _i, _i, _i, _d, _d, _p, _z, _p, _p], _i),
    "kle_2d_cgc_work_doubles": ([_i, _i, _i], _z),
    "kle_2d_cgc_f64": ([_p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _i, _d, _p, _p, _p, _p, _p, _p, _z, _p], _i),
    "kle_2d_fgr_krylov_f64": ([_p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _d, _d, _d, _d, _d, _i, _p, _p, _p,
                               _p], _i),
    "kle_2d_sweep_krylov_f64": ([_p, _p, _p, _p, _i, _i, _i, _i, _d, _d, _d, _i, _p, _p, _p], _i),
    "kle_2d_cgc_krylov_work_doubles": ([_i, _i, _i], _z),
    "kle_2d_cgc_krylov_f64": ([_p, _p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _i, _d, _p, _p, _p, _p, _p, _d,
                               _d, _i, _p, _z, _p, _p], _i),
    "kle_gpc_basis_f64": ([_p, _i, _i, _i, _i, _p, _p, _i, _p, _p, _p], _i),
    "kle_gpc_eval_f64": ([_p, _i, _i, _p, _p, _i, _p, _p], _i),
    "kle_gemm_f64": ([_p, _p, _p, _p, _i, _i, _i, _i, _p], _i),
    "kle_sub_row_f64": ([_p, _p, _p, _i, _i, _p], _i),
    "kle_col_sum_scratch_bytes": ([_i, _i], _z),
    "kle_col_sum_f64": ([_p, _i, _i, _p, _p, _p, _p], _i),
    "kle_axpby_f64": ([_p, _p, _p, _d, _d, _z, _p], _i),
}

EXPORTED = tuple(_SIGS)


def library_path() -> Path:
    return Path(os.environ.get("KLE_B200_LIB", _LIB_PATH))


def load():
    """Load (once) and return the CDLL; raises DeviceError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        raise DeviceError(
            f"{path} not found: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2510_26180_b200/csrc)"
        )
    lib = C.CDLL(str(path))
    for name, (argt, rest) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = argt
        fn.restype = rest
    if lib.kle_abi_version() != 1:
        raise DeviceError("libkle_b200.so ABI version mismatch")
    _lib = lib
    return lib


def call(name: str, *args) -> int:
    """Invoke an entry point; a non-zero status raises DeviceError."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if _SIGS[name][1] is _i and name.endswith("_f64") and rc != 0:
        msg = lib.kle_last_error().decode(errors="replace")
        raise DeviceError(f"{name} failed (code {rc}): {msg}")
    return rc


def query(name: str, *args):
    return getattr(load(), name)(*args)
