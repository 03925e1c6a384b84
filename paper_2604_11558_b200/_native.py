"""ctypes binding of libcurvigpu.so (C ABI in include/curvigpu.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2604_11558_b200.build``).  There is no fallback: if the
shared object is missing or a call fails, an exception is raised.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libcurvigpu.so"

CG_OK = 0
CG_EINVAL = -1
CG_ECUDA = -2
CG_EUNSUPPORTED = -3

GEOMETRY_CODES = {"disk": 0, "sphere": 1, "ball": 2, "cylinder": 3}
CG_OPT_THETA_FFT = 1


class EngineError(RuntimeError):
    """A libcurvigpu call failed (message from cg_last_error)."""


class cg_desc(ctypes.Structure):
    _dp = ctypes.POINTER(ctypes.c_double)
    _fields_ = [
        ("geometry", ctypes.c_int),
        ("n", ctypes.c_int * 3),
        ("batch", ctypes.c_int),
        ("ncomp", ctypes.c_int),
        ("tau", ctypes.c_double),
        ("coeff", _dp),
        ("rho_bands", _dp),
        ("phi_bands", _dp),
        ("z_bands", _dp),
        ("theta_stencil", _dp),
        ("d_rho", _dp),
        ("d_phi", _dp),
        ("Q_theta", _dp),
        ("phi1_rho", _dp),
        ("phi1_phi", _dp),
        ("phi1_z", _dp),
        ("V_phi", _dp),
        ("Vinv_phi", _dp),
        ("Phi", _dp),
        ("Phi_outer", _dp),
        ("kinetics", ctypes.c_int),
        ("nparams", ctypes.c_int),
        ("kin_params", _dp),
        ("lift", _dp),
        ("options", ctypes.c_int),
        ("ops_per_run", ctypes.c_int),
    ]


_lib = None

EXPORTS = (
    "cg_plan_create",
    "cg_plan_destroy",
    "cg_plan_state_elems",
    "cg_apply_diffusion",
    "cg_kinetics",
    "cg_step",
    "cg_run",
    "cg_last_error",
    "cg_version",
    "cg_rng_seed",
    "cg_rng_next",
    "cg_rng_uniform",
    "cg_rng_normal",
    "cg_plan_stage_count",
    "cg_plan_stage_info",
    "cg_run_stage",
    "cg_plan_step_kernels",
    "cg_plan_copy_workspace",
    "cg_plan_check_redzones",
    "cg_step_guarded",
    "cg_plan_set_step",
    "cg_coupling_create",
    "cg_coupling_destroy",
    "cg_coupled_kinetics",
    "cg_coupled_run",
    "cg_weighted_sums_scratch",
    "cg_weighted_sums",
    "cg_product_create",
    "cg_product_apply",
    "cg_product_destroy",
    "cg_hadamard",
    "cg_setup_eig_tridiag",
    "cg_setup_phi1_matrix",
    "cg_setup_phi1_outer",
    "cg_setup_phi1",
)

CG_BS_BALL = 1
CG_BS_CYLINDER = 2


class cg_coupling_desc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("nb", ctypes.c_int * 3),
        ("ns", ctypes.c_int * 2),
        ("params", ctypes.POINTER(ctypes.c_double)),
        ("nparams", ctypes.c_int),
        ("geom", ctypes.c_double * 2),
        ("lift", ctypes.c_double * 4),
    ]


def lib():
    """Load (once) and return the shared library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("CURVIGPU_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise EngineError(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    L = ctypes.CDLL(path)
    vp = ctypes.c_void_p
    dp = ctypes.POINTER(ctypes.c_double)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    L.cg_plan_create.argtypes = [ctypes.POINTER(cg_desc), ctypes.POINTER(vp)]
    L.cg_plan_create.restype = ctypes.c_int
    L.cg_plan_destroy.argtypes = [vp]
    L.cg_plan_destroy.restype = None
    L.cg_plan_state_elems.argtypes = [vp]
    L.cg_plan_state_elems.restype = ctypes.c_longlong
    L.cg_apply_diffusion.argtypes = [vp, vp, vp, vp]
    L.cg_apply_diffusion.restype = ctypes.c_int
    L.cg_kinetics.argtypes = [vp, vp, vp, vp]
    L.cg_kinetics.restype = ctypes.c_int
    L.cg_step.argtypes = [vp, vp, vp, vp, vp]
    L.cg_step.restype = ctypes.c_int
    L.cg_run.argtypes = [vp, vp, ctypes.c_longlong, ctypes.c_longlong, vp, vp]
    L.cg_run.restype = ctypes.c_int
    L.cg_last_error.argtypes = []
    L.cg_last_error.restype = ctypes.c_char_p
    L.cg_version.argtypes = []
    L.cg_version.restype = ctypes.c_int
    L.cg_rng_seed.argtypes = [ctypes.c_uint64, u64p]
    L.cg_rng_seed.restype = None
    L.cg_rng_next.argtypes = [u64p, ctypes.c_longlong, u64p]
    L.cg_rng_next.restype = None
    L.cg_rng_uniform.argtypes = [u64p, ctypes.c_longlong, ctypes.c_double, ctypes.c_double, dp]
    L.cg_rng_uniform.restype = None
    L.cg_rng_normal.argtypes = [u64p, ctypes.c_longlong, ctypes.c_double, dp]
    L.cg_rng_normal.restype = None
    L.cg_plan_stage_count.argtypes = [vp]
    L.cg_plan_stage_count.restype = ctypes.c_int
    L.cg_plan_stage_info.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong),
                                     ctypes.POINTER(ctypes.c_longlong)]
    L.cg_plan_stage_info.restype = ctypes.c_int
    L.cg_run_stage.argtypes = [vp, ctypes.c_int, vp, vp, vp, vp]
    L.cg_run_stage.restype = ctypes.c_int
    L.cg_plan_step_kernels.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.c_int]
    L.cg_plan_step_kernels.restype = ctypes.c_int
    L.cg_plan_copy_workspace.argtypes = [vp, ctypes.c_int, vp, vp]
    L.cg_plan_copy_workspace.restype = ctypes.c_int
    L.cg_plan_check_redzones.argtypes = [vp]
    L.cg_plan_check_redzones.restype = ctypes.c_longlong
    L.cg_step_guarded.argtypes = [vp, vp, vp, vp, vp, vp]
    L.cg_step_guarded.restype = ctypes.c_int
    L.cg_plan_set_step.argtypes = [vp, ctypes.c_longlong, vp]
    L.cg_plan_set_step.restype = ctypes.c_int
    L.cg_coupling_create.argtypes = [ctypes.POINTER(cg_coupling_desc), ctypes.POINTER(vp)]
    L.cg_coupling_create.restype = ctypes.c_int
    L.cg_coupling_destroy.argtypes = [vp]
    L.cg_coupling_destroy.restype = None
    L.cg_coupled_kinetics.argtypes = [vp, vp, vp, vp, vp, vp]
    L.cg_coupled_kinetics.restype = ctypes.c_int
    L.cg_coupled_run.argtypes = [vp, vp, vp, vp, vp, ctypes.c_longlong, ctypes.c_longlong, vp, vp]
    L.cg_coupled_run.restype = ctypes.c_int
    L.cg_weighted_sums_scratch.argtypes = [ctypes.c_longlong, ctypes.c_longlong]
    L.cg_weighted_sums_scratch.restype = ctypes.c_longlong
    L.cg_weighted_sums.argtypes = [vp, ctypes.c_longlong, ctypes.c_longlong, vp, ctypes.c_int, vp, vp, vp,
                                   ctypes.c_longlong, vp]
    L.cg_weighted_sums.restype = ctypes.c_int
    ci = ctypes.c_int
    L.cg_product_create.argtypes = [ci, ci, ctypes.POINTER(ci), dp, ctypes.POINTER(vp)]
    L.cg_product_create.restype = ci
    L.cg_product_apply.argtypes = [vp, vp, vp, vp]
    L.cg_product_apply.restype = ci
    L.cg_product_destroy.argtypes = [vp]
    L.cg_product_destroy.restype = None
    L.cg_hadamard.argtypes = [vp, vp, vp, ctypes.c_longlong, vp]
    L.cg_hadamard.restype = ci
    L.cg_setup_eig_tridiag.argtypes = [ci, ci, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.cg_setup_eig_tridiag.restype = ci
    L.cg_setup_phi1_matrix.argtypes = [ci, ci, vp, vp, vp, vp, vp, vp, vp]
    L.cg_setup_phi1_matrix.restype = ci
    L.cg_setup_phi1_outer.argtypes = [ci, ci, ci, ci, vp, vp, vp, vp, vp, vp]
    L.cg_setup_phi1_outer.restype = ci
    L.cg_setup_phi1.argtypes = [ctypes.c_longlong, vp, vp, vp]
    L.cg_setup_phi1.restype = ci
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != CG_OK:
        msg = lib().cg_last_error().decode(errors="replace")
        if rc == CG_EINVAL:
            raise ValueError(f"{what}: {msg}")
        if rc == CG_EUNSUPPORTED:
            raise NotImplementedError(f"{what}: {msg}")
        raise EngineError(f"{what} failed ({rc}): {msg}")


def dptr(arr):
    """ctypes double* for a C-contiguous float64 numpy array (or None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
