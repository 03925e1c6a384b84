"""The C-ABI library loads and exports every entry point include/curvigpu.h
declares; the sm_100a cubin carries DMMA and TMA instructions.  CPU only:
no compute call is made here."""

import re
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2604_11558_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "curvigpu.h").read_text()
    return sorted(set(re.findall(r"\b(cg_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_api():
    syms = declared_symbols()
    assert set(syms) == set(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym
    assert lib.cg_version() == 1


def test_plan_create_rejects_bad_descriptors_without_touching_the_gpu():
    import ctypes

    lib = _native.lib()
    d = _native.cg_desc()
    d.geometry = 7
    h = ctypes.c_void_p()
    rc = lib.cg_plan_create(ctypes.byref(d), ctypes.byref(h))
    assert rc == _native.CG_EINVAL
    assert b"geometry" in lib.cg_last_error()
    d.geometry = 0
    d.n[0], d.n[1], d.n[2] = 64, 127, 1
    d.batch, d.ncomp = 1, 3  # built-in kinetics are two-species
    d.kinetics = 1
    rc = lib.cg_plan_create(ctypes.byref(d), ctypes.byref(h))
    assert rc == _native.CG_EUNSUPPORTED
    with pytest.raises(NotImplementedError):
        _native.check(rc, "cg_plan_create")


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not Path("/usr/local/cuda/bin/cuobjdump").exists(),
                    reason="cuobjdump missing")
def test_cubin_is_sm100a_with_dmma_and_tma():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([tool, "-sass", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    assert "DMMA.8x8x4" in sass
    assert "UTMALDG" in sass
