"""The reference-facing side of the drop-in (INTEGRATION.md Option B).

What a ``curvipat`` maintainer's ``device="b200"`` switch calls: the
engine's entry points with the engine's own exceptions re-raised as the
reference's classes, so every caller that catches them keeps working --
``cmd_run``'s partial-output handler (``except DivergenceError``,
src/cli.py:235-240) and ``main``'s exit codes 3 (DivergenceError) and 4
(NumericalFailure) (src/cli.py:494-499).

The reference is never imported here: the classes are looked up in
``sys.modules``, i.e. only when the caller (curvipat itself) has loaded
them.  Without curvipat in the process the engine's exceptions pass through
unchanged (they carry the same fields: ``DivergenceError.step``).
"""

from __future__ import annotations

import contextlib
import sys

from . import integrators as _eng
from .operators import NumericalFailure as _EngineNumericalFailure


def reference_error_types():
    """(curvipat DivergenceError, curvipat NumericalFailure), each None when
    that reference module is not loaded in this process."""
    integ = sys.modules.get("curvipat.integrators")
    ops = sys.modules.get("curvipat.operators")
    return getattr(integ, "DivergenceError", None), getattr(ops, "NumericalFailure", None)


def translate(exc: BaseException) -> BaseException:
    """The reference-class equivalent of an engine exception (same message,
    same ``step``), or ``exc`` itself when there is none."""
    ref_div, ref_num = reference_error_types()
    if isinstance(exc, _eng.DivergenceError) and ref_div is not None and not isinstance(exc, ref_div):
        return ref_div(str(exc), step=exc.step)
    if isinstance(exc, _EngineNumericalFailure) and ref_num is not None and not isinstance(exc, ref_num):
        return ref_num(str(exc))
    return exc


@contextlib.contextmanager
def reference_errors():
    """Re-raise engine DivergenceError / NumericalFailure raised inside the
    block as curvipat's own classes (chained to the engine's)."""
    try:
        yield
    except (_eng.DivergenceError, _EngineNumericalFailure) as exc:
        ref = translate(exc)
        if ref is exc:
            raise
        raise ref from exc


def run_simulation(system, m, t_star, *, record_every=None, diagnostics=None, sample_hook=None,
                   method="split", **kw):
    """curvipat.integrators.run_simulation (src/integrators.py:370-430) on
    the B200 engine, raising the reference's exception classes."""
    with reference_errors():
        return _eng.run_simulation(system, m, t_star, record_every=record_every, diagnostics=diagnostics,
                                   sample_hook=sample_hook, method=method, **kw)


def prepare(base, tau):
    """curvipat.integrators.prepare (src/integrators.py:130-173), host setup."""
    with reference_errors():
        return _eng.prepare(base, tau)


def step_split(ops, W, G):
    """curvipat.integrators.step_split (src/integrators.py:247-249) on the GPU."""
    with reference_errors():
        return _eng.step_split(ops, W, G)


def apply_diffusion(ops, W):
    """curvipat.integrators.apply_diffusion (src/integrators.py:176-199) on the GPU."""
    with reference_errors():
        return _eng.apply_diffusion(ops, W)
