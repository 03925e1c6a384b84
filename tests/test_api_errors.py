"""Error behaviour of the reference-shaped entry points, mirroring the
reference's own checks (tests/test_integrators.py:105-108 and :347-354 of
the reference suite; src/integrators.py:178-179, :388-393).  Every error
here is raised before any device work, so these run without a GPU."""

import numpy as np
import pytest

from paper_2604_11558_b200 import models
from paper_2604_11558_b200.integrators import (STEPPERS, ComponentOps, Geometry, apply_diffusion, prepare,
                                               run_simulation, step_split)
from paper_2604_11558_b200.ensemble import run_ensemble

DIMS = {"n_rho": 4, "n_theta": 6}


def _disk_ops():
    system = models.build_system("bvam_disk", DIMS, seed=4)
    return system, prepare(system.components[0].ops, 0.1)


def test_apply_diffusion_shape_error():
    _, ops = _disk_ops()
    with pytest.raises(ValueError):
        apply_diffusion(ops, np.zeros((5, 4)))


def test_step_split_shape_errors():
    _, ops = _disk_ops()
    good = np.zeros(ops.shape)
    with pytest.raises(ValueError):
        step_split(ops, np.zeros((5, 4)), good)
    with pytest.raises(ValueError):
        step_split(ops, good, np.zeros((ops.shape[0] + 1, ops.shape[1])))


def test_geometry_stepper_rejects_other_geometry():
    _, ops = _disk_ops()
    good = np.zeros(ops.shape)
    with pytest.raises(ValueError):
        STEPPERS[Geometry.SPHERE](ops, good, good)


def test_run_simulation_validates_inputs():
    system = models.build_system("bvam_disk", DIMS, seed=4)
    with pytest.raises(ValueError):
        run_simulation(system, 0, 1.0)
    with pytest.raises(ValueError):
        run_simulation(system, 5, -1.0)
    with pytest.raises(ValueError):
        run_simulation(system, 5, 1.0, method="leapfrog")
    # the reference's forward Euler comparison path is out of scope: it fails loudly
    with pytest.raises(NotImplementedError):
        run_simulation(system, 5, 1.0, method="forward_euler")


def test_run_ensemble_validates_inputs():
    system = models.build_system("bvam_disk", DIMS, seed=4)
    with pytest.raises(ValueError):
        run_ensemble([system], 0, 1.0)
    with pytest.raises(ValueError):
        run_ensemble([system], 5, 0.0)
    with pytest.raises(ValueError):
        run_ensemble([], 5, 1.0)


def test_inputs_are_not_mutated_by_failed_calls():
    system = models.build_system("bvam_disk", DIMS, seed=4)
    before = [c.initial.copy() for c in system.components]
    with pytest.raises(ValueError):
        run_simulation(system, 0, 1.0)
    for c, b in zip(system.components, before):
        assert np.array_equal(c.initial, b)


def test_component_ops_is_frozen():
    system = models.build_system("bvam_disk", DIMS, seed=4)
    ops = system.components[0].ops
    assert isinstance(ops, ComponentOps) or hasattr(ops, "geometry")
    with pytest.raises(Exception):
        ops.coeff = 2.0
