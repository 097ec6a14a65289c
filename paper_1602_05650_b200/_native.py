"""ctypes binding of libsf_b200.so (the C ABI declared in include/sf_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every device entry point raises NativeUnavailable.
"""

import ctypes
import os

from .build import LIB

SF_OK = 0
SF_MODE_FP64 = 0
SF_MODE_FP32C = 1
SF_MODE_FP64_DIRECT = 2


class NativeUnavailable(RuntimeError):
    """The sm_100a library could not be loaded (not built, or no GPU)."""


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, fn, code, msg):
        super().__init__(f"{fn} failed with status {code}: {msg}")
        self.code = code


_D = ctypes.c_double
_I64 = ctypes.c_int64
_I = ctypes.c_int
_P = ctypes.c_void_p

# name -> argtypes (all return int status)
_SIGNATURES = {
    "sf_abi_version": [],
    "sf_device_sm_count": [],
    "sf_stokeslet_sum": [_P, _P, _I64, _P, _P, _I64, _P, _D, _P, _P, _P],
    "sf_doublet_sum": [_P, _P, _I64, _P, _P, _I64, _P, _D, _P, _P, _P],
    "sf_sbt_pair": [_P, _P, _I64, _P, _P, _I64, _P, _P, _D, _I, _P, _P, _P],
    "sf_stresslet_sum": [_P, _P, _I64, _P, _P, _I64, _P, _P, _D, _P, _P, _P],
    "sf_stresslet_sum_subtracted": [_P, _P, _P, _P, _I64, _D, _P, _P],
    "sf_stresslet_sum_subtracted_partial": [_P, _P, _P, _P, _I64, _D, _I, _I, _P, _P],
    "sf_stresslet_rowsum": [_P, _P, _P, _I64, _D, _P, _P],
    "sf_kdelta_build_batched": [_P, _P, _P, _P, _P, _I64, _I64, _P, _D, _P, _P],
    "sf_self_apply_batched": [_P, _P, _P, _D, _P, _I64, _I64, _I, _P, _P],
    "sf_near_apply": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P],
    "sf_fiber_geometry_batched": [_P, _I64, _I64, _P, _P, _P, _D, _P, _P, _P, _P, _P, _P, _P,
                                  _P],
    "sf_fiber_hi_apply": [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _D, _I, _P, _P, _P, _D, _P,
                          _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "sf_pair_split": [_I64, _I64],
    "sf_tree_stokeslet": [_P, _P, _I64, _P, _P, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _I64,
                          _D, _D, _D, _P, _P, _P],
    "sf_tree_work_doubles": [_I64],
    "sf_sym_shard_pairs": [_I64, _I64, _I, _I],
    "sf_sym_launch_count": [_I64, _I64, _I, _I, _I],
    "sf_sym_set_waves": [_I64, _I],
    "sf_workspace_bytes": [],
    "sf_workspace_release": [],
    "sf_sbt_symmetric_partial": [_P, _P, _I64, _I64, _P, _P, _P, _D, _I, _I, _I, _P, _P, _P],
    "sf_sbt_symmetric_tasks": [_P, _P, _I64, _I64, _P, _P, _P, _D, _I, _I64, _I64, _P, _P, _P],
    "sf_sym_task_count": [_I64, _I64, _I],
    "sf_sym_unit_size": [_I64, _I64, _I],
    "sf_sym_task_costs": [_P, _P, _I64, _I64, _I, _D, _D, _P, _P],
    "sf_sym_range_pairs": [_I64, _I64, _I, _I64, _I64],
    "sf_sym_range_launch_count": [_I64, _I64, _I, _I64, _I64],
    "sf_hi_apply": [_P, _P, _P, _P, _P, _P, _P, _P],
    "sf_fiber_dpow": [_P, _P, _I64, _I64, _P, _P],
    "sf_near_search": [_P, _P, _I64, _P, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P],
    "sf_near_surface_weights": [_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _I, _I64, _P, _P, _P, _P,
                                _P, _P, _P, _D, _P, _P, _P],
    "sf_near_fiber_weights": [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _D, _I,
                              _P, _P, _P],
    "sf_fiber_forces": [_P, _P, _I, _P, _P],
    "sf_particle_wrenches": [_P, _P, _P, _I, _P, _P, _P],
    "sf_fiber_rows": [_P, _P, _P, _P, _I, _P, _P],
    "sf_fiber_self_blocks": [_P, _P, _P],
    "sf_block_lu": [_P, _I64, _I64, _P, _P, _P, _P, _P],
    "sf_block_solve": [_P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P],
    "sf_precond_apply": [_P, _P, _P, _P, _I64, _I64, _I64, _P, _I64, _P, _P, _P],
    "sf_surface_rows": [_I, _P, _P, _P, _I64, _P, _D, _P, _P, _P, _D, _P, _P, _P, _P],
    "sf_wrench_flow": [_P, _I64, _P, _P, _D, _P, _P],
    "sf_dot": [_P, _P, _I64, _P, _P, _I, _P],
    "sf_axpy_dev": [_P, _D, _I, _P, _P, _I64, _P],
    "sf_combine": [_P, _I64, _I, _P, _P, _I64, _P],
    "sf_gmres_mgs": [_P, _I64, _I, _P, _I64, _P, _I, _P, _P],
    "sf_gmres_state_doubles": [_I, _I],
    "sf_gmres_reset": [_P, _I, _I, _D, _D, _P],
    "sf_gmres_cycle": [_P, _I, _P, _P, _P, _I64, _P],
    "sf_gmres_givens": [_P, _P, _I, _I, _P, _P],
    "sf_gmres_mgs_dk": [_P, _I64, _P, _P, _I64, _P, _I, _P, _P],
    "sf_gmres_update": [_P, _I64, _P, _I, _P, _I64, _P],
    "sf_host_stokeslet_sum": [_P, _P, _I64, _P, _P, _I64, _P, _D, _P, _P],
    "sf_host_doublet_sum": [_P, _P, _I64, _P, _P, _I64, _P, _D, _P, _P],
    "sf_host_sbt_pair": [_P, _P, _I64, _P, _P, _I64, _P, _P, _D, _I, _P, _P],
    "sf_host_stresslet_sum": [_P, _P, _I64, _P, _P, _I64, _P, _P, _D, _P, _P],
    "sf_host_stresslet_sum_subtracted": [_P, _P, _P, _P, _I64, _D, _P],
    "sf_host_stresslet_rowsum": [_P, _P, _P, _I64, _D, _P],
    "sf_host_kdelta_matrix": [_P, _P, _P, _P, _P, _I64, _D, _D, _P],
    "sf_dfma_peak": [_I64, _P, _P],
}

_lib = None
_device_ok = False


class FiberSys(ctypes.Structure):
    """Mirror of sf_fiber_sys (include/sf_b200.h)."""
    _fields_ = [
        ("nf", _I64), ("n", _I64), ("D", _P), ("nodes", _P), ("Dpow", _P), ("X", _P),
        ("tang", _P), ("s_alpha", _P), ("L", _P), ("Ldot", _P), ("E", _P), ("c_log", _P),
        ("c_two", _D), ("K", _P), ("f_ext", _P), ("bc_kind", _P), ("bc_par", _P),
        ("bc_body", _P), ("np", _I64), ("pcenter", _P), ("p_uoff", _P), ("fib_off", _I64),
        ("dt", _D), ("mu", _D), ("u_off", _P), ("pt_off", _P),
    ]


class HiLayout(ctypes.Structure):
    """Mirror of sf_hi_layout (include/sf_b200.h)."""
    _fields_ = [
        ("trg", _P), ("tgrp", _P), ("nt", _I64),
        ("fsrc", _P), ("fgrp", _P), ("fw", _P), ("fdcoef", _P), ("nfs", _I64),
        ("ssrc", _P), ("snrm", _P), ("sw", _P), ("sgrp", _P), ("nss", _I64),
        ("pcenter", _P), ("pgrp", _P), ("np", _I64),
        ("near_row_ptr", _P), ("near_rows", _P), ("near_w_off", _P), ("near_x_off", _P),
        ("near_x_len", _P), ("near_nrows", _I64), ("near_W", _P),
        ("mu", _D), ("mode", _I), ("fiber_target_off", _I64), ("fiber_group_size", _I64),
    ]


def exported_symbols():
    return sorted(_SIGNATURES) + ["sf_last_error"]


def load(require_device=False):
    """Load the library (cached).  require_device also checks for a GPU."""
    global _lib, _device_ok
    if _lib is None:
        if not os.path.exists(LIB):
            raise NativeUnavailable(
                f"{LIB} is not built; run `python -m paper_1602_05650_b200.build`")
        lib = ctypes.CDLL(LIB)
        for name, argtypes in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _I
        lib.sf_sym_shard_pairs.restype = ctypes.c_int64
        lib.sf_sym_launch_count.restype = ctypes.c_int64
        lib.sf_sym_task_count.restype = ctypes.c_int64
        lib.sf_sym_unit_size.restype = ctypes.c_int64
        lib.sf_sym_range_pairs.restype = ctypes.c_int64
        lib.sf_sym_range_launch_count.restype = ctypes.c_int64
        lib.sf_workspace_bytes.restype = ctypes.c_int64
        lib.sf_gmres_state_doubles.restype = ctypes.c_int64
        lib.sf_tree_work_doubles.restype = ctypes.c_int64
        lib.sf_last_error.argtypes = []
        lib.sf_last_error.restype = ctypes.c_char_p
        _lib = lib
    if require_device and not _device_ok:
        if _lib.sf_device_sm_count() <= 0:
            raise NativeUnavailable("no CUDA device visible to libsf_b200")
        _device_ok = True
    return _lib


def call(name, *args):
    lib = load(require_device=True)
    rc = getattr(lib, name)(*args)
    if rc != SF_OK:
        raise NativeError(name, rc, lib.sf_last_error().decode(errors="replace"))
    return rc
