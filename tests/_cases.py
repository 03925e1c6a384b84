"""Named single-component cases shared by the parity tests; they mirror
``_bases()`` in tests/golden/make_golden.py (reference side)."""

from __future__ import annotations

from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import operators as op
from paper_2604_11558_b200.integrators import ComponentOps, Geometry

CASES = [
    "disk_4x4",
    "sphere_4x4",
    "ball_3x4x4",
    "cylinder_3x4x4",
    "disk_20x36",
    "adisk_33x64",
    "sphere_40x34",
    "ball_12x10x18",
    "cylinder_9x20x24",
    "cylinderD_6x8x10",
    # odd contiguous (last) axes: the reference's own test bases
    # (tests/test_integrators.py:38 ball_base(3, 4, 3); tests/test_models.py:183
    # dib_sphere (8, 5)) and odd theta on the disk
    "ball_3x4x3",
    "sphere_8x5",
    "disk_5x7",
    "cylinder_3x4x5",
    "sphere_7x9",
]


def engine_base(name):
    if name == "disk_4x4":
        return ComponentOps(Geometry.DISK, 0.7, rho=op.build_rho(2, 4, 1.0), theta=op.build_theta(4))
    if name == "sphere_4x4":
        return ComponentOps(Geometry.SPHERE, 0.9, theta=op.build_theta(4), phi=op.build_phi_op(4)[0])
    if name == "ball_3x4x4":
        return ComponentOps(Geometry.BALL, 1.1, rho=op.build_rho(3, 3, 1.0), theta=op.build_theta(4),
                            phi=op.build_phi_op(4)[0])
    if name == "cylinder_3x4x4":
        return ComponentOps(Geometry.CYLINDER, 0.8, rho=op.build_rho(2, 3, 1.0), theta=op.build_theta(4),
                            z=op.build_z(4, 1.0))
    if name == "disk_20x36":
        return ComponentOps(Geometry.DISK, 1.3, rho=op.build_rho(2, 20, 1.0), theta=op.build_theta(36))
    if name == "adisk_33x64":
        lam = op.build_lambda(33, 1.0, -1.95)
        return ComponentOps(Geometry.DISK, 10.0, rho=lam, theta=op.build_theta(64),
                            rho_weights=op.DiagonalWeights(lam.grid ** (-2.0 + 1.95)))
    if name == "sphere_40x34":
        return ComponentOps(Geometry.SPHERE, 0.08, theta=op.build_theta(40), phi=op.build_phi_op(34)[0])
    if name == "ball_12x10x18":
        return ComponentOps(Geometry.BALL, 0.516, rho=op.build_rho(3, 12, 1.0), theta=op.build_theta(10),
                            phi=op.build_phi_op(18)[0])
    if name == "cylinder_9x20x24":
        return ComponentOps(Geometry.CYLINDER, 2e-2, rho=op.build_rho(2, 9, 1.0), theta=op.build_theta(20),
                            z=op.build_z_neumann(24, 2.0))
    if name == "cylinderD_6x8x10":
        return ComponentOps(Geometry.CYLINDER, 0.3, rho=op.build_rho(2, 6, 1.0), theta=op.build_theta(8),
                            z=op.build_z(10, 1.5))
    if name == "ball_3x4x3":
        return ComponentOps(Geometry.BALL, 1.1, rho=op.build_rho(3, 3, 1.0), theta=op.build_theta(4),
                            phi=op.build_phi_op(3)[0])
    if name == "sphere_8x5":
        return ComponentOps(Geometry.SPHERE, 0.9, theta=op.build_theta(8), phi=op.build_phi_op(5)[0])
    if name == "disk_5x7":
        return ComponentOps(Geometry.DISK, 0.7, rho=op.build_rho(2, 5, 1.0), theta=op.build_theta(7))
    if name == "cylinder_3x4x5":
        return ComponentOps(Geometry.CYLINDER, 0.8, rho=op.build_rho(2, 3, 1.0), theta=op.build_theta(4),
                            z=op.build_z(5, 1.0))
    if name == "sphere_7x9":
        return ComponentOps(Geometry.SPHERE, 0.3, theta=op.build_theta(7), phi=op.build_phi_op(9)[0])
    raise KeyError(name)


def oracle_comp(name):
    if name == "disk_4x4":
        return orc.Comp("w", "disk", 0.7, rho=orc.radial_stencil(2, 4, 1.0), theta=orc.theta_stencil(4))
    if name == "sphere_4x4":
        return orc.Comp("w", "sphere", 0.9, theta=orc.theta_stencil(4), phi=orc.polar_stencil(4))
    if name == "ball_3x4x4":
        return orc.Comp("w", "ball", 1.1, rho=orc.radial_stencil(3, 3, 1.0), theta=orc.theta_stencil(4),
                        phi=orc.polar_stencil(4))
    if name == "cylinder_3x4x4":
        return orc.Comp("w", "cylinder", 0.8, rho=orc.radial_stencil(2, 3, 1.0), theta=orc.theta_stencil(4),
                        z=orc.axial_stencil_nd(4, 1.0))
    if name == "disk_20x36":
        return orc.Comp("w", "disk", 1.3, rho=orc.radial_stencil(2, 20, 1.0), theta=orc.theta_stencil(36))
    if name == "adisk_33x64":
        lam = orc.anomalous_stencil(33, 1.0, -1.95)
        return orc.Comp("w", "disk", 10.0, rho=lam, theta=orc.theta_stencil(64),
                        rho_weights=lam.grid ** (-2.0 + 1.95))
    if name == "sphere_40x34":
        return orc.Comp("w", "sphere", 0.08, theta=orc.theta_stencil(40), phi=orc.polar_stencil(34))
    if name == "ball_12x10x18":
        return orc.Comp("w", "ball", 0.516, rho=orc.radial_stencil(3, 12, 1.0), theta=orc.theta_stencil(10),
                        phi=orc.polar_stencil(18))
    if name == "cylinder_9x20x24":
        return orc.Comp("w", "cylinder", 2e-2, rho=orc.radial_stencil(2, 9, 1.0), theta=orc.theta_stencil(20),
                        z=orc.axial_stencil_nn(24, 2.0))
    if name == "cylinderD_6x8x10":
        return orc.Comp("w", "cylinder", 0.3, rho=orc.radial_stencil(2, 6, 1.0), theta=orc.theta_stencil(8),
                        z=orc.axial_stencil_nd(10, 1.5))
    if name == "ball_3x4x3":
        return orc.Comp("w", "ball", 1.1, rho=orc.radial_stencil(3, 3, 1.0), theta=orc.theta_stencil(4),
                        phi=orc.polar_stencil(3))
    if name == "sphere_8x5":
        return orc.Comp("w", "sphere", 0.9, theta=orc.theta_stencil(8), phi=orc.polar_stencil(5))
    if name == "disk_5x7":
        return orc.Comp("w", "disk", 0.7, rho=orc.radial_stencil(2, 5, 1.0), theta=orc.theta_stencil(7))
    if name == "cylinder_3x4x5":
        return orc.Comp("w", "cylinder", 0.8, rho=orc.radial_stencil(2, 3, 1.0), theta=orc.theta_stencil(4),
                        z=orc.axial_stencil_nd(5, 1.0))
    if name == "sphere_7x9":
        return orc.Comp("w", "sphere", 0.3, theta=orc.theta_stencil(7), phi=orc.polar_stencil(9))
    raise KeyError(name)
