"""On-device setup: ``prepare_device`` is a batched drop-in for
``integrators.prepare`` (reference ``prepare``, integrators.py:130-173) that
evaluates the per-operator work on the GPU through ``libcurvigpu``:

- ``eig_tridiag`` (operators.py:357-382; LAPACK through scipy in the
  reference) -> ``cg_setup_eig_tridiag``: symmetriser + implicit-shift QL, one
  CTA per distinct operator;
- ``phi1_matrix`` (phifun.py:68-71) -> ``cg_setup_phi1_matrix``: one launch
  for every (run, component) of an axis;
- ``phi1_outer`` (phifun.py:52-65) -> ``cg_setup_phi1_outer``: the Phi tensors
  of every (run, component) in one launch.

It is meant for heterogeneous ensembles (``SplitPlan(ops_per_run=True)``),
where every run brings its own coefficients or domain sizes: the host path
evaluates 2 x B eigenproblems / phi1 tables one after the other, the device
path evaluates them all at once.  The closed-form pieces (the periodic
Fourier basis ``eig_theta``, metric weights, dense operator copies kept for
API parity) stay on the host, as does the final hand-over: the tables come
back as NumPy arrays inside ordinary ``GeometryOps`` objects, which
``SplitPlan`` uploads in its own layouts.  There is no CPU fallback: without
the CUDA library or a GPU the call raises.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .integrators import GeometryOps, _cached, _geometry_name, _op_key, _rho_weights
from .operators import EigenFactorization, NumericalFailure, eig_theta
from .phifun import PhiTensor


_MAX_SETS = 32768  # sets per cg_setup_phi1_* launch (the C ABI takes up to 65535)


def _stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).cuda()


class _EigBatch:
    """Distinct tridiagonal operators of one extent n, solved in one launch."""

    def __init__(self, n: int):
        self.n = n
        self.index: dict = {}
        self.ops: list = []

    def add(self, op) -> int:
        key = _op_key(op)
        hit = self.index.get(key)
        if hit is None:
            hit = self.index[key] = len(self.ops)
            self.ops.append(op)
        return hit

    def solve(self):
        import torch

        n, m = self.n, len(self.ops)
        for op in self.ops:
            if np.any(np.asarray(op.b) <= 0) or np.any(np.asarray(op.c) <= 0):
                raise ValueError("symmetrization needs strictly positive off-diagonals")
        a = _dev(np.stack([np.asarray(op.a, dtype=float) for op in self.ops]))
        b = _dev(np.stack([np.asarray(op.b, dtype=float) for op in self.ops]))
        c = _dev(np.stack([np.asarray(op.c, dtype=float) for op in self.ops]))
        self.lam = torch.empty((m, n), dtype=torch.float64, device="cuda")
        self.Qt = torch.empty((m, n, n), dtype=torch.float64, device="cuda")
        self.xi = torch.empty((m, n), dtype=torch.float64, device="cuda")
        work = torch.empty((m, n, n), dtype=torch.float64, device="cuda")
        self.status = torch.full((m,), -1, dtype=torch.int32, device="cuda")
        _native.check(_native.lib().cg_setup_eig_tridiag(m, n, a.data_ptr(), b.data_ptr(), c.data_ptr(),
                                                         self.lam.data_ptr(), self.Qt.data_ptr(), self.xi.data_ptr(),
                                                         work.data_ptr(), self.status.data_ptr(), _stream()),
                      "cg_setup_eig_tridiag")
        return self

    def check(self):
        st = self.status.cpu().numpy()
        if np.any(st == 2):
            raise ValueError("symmetrization needs strictly positive off-diagonals")
        if np.any(st != 0):
            raise NumericalFailure(f"tridiagonal eigensolver failed: QL iteration did not converge "
                                   f"(operator {int(np.flatnonzero(st != 0)[0])} of {len(st)})")

    def factorizations(self) -> list[EigenFactorization]:
        lam = self.lam.cpu().numpy()
        Q = self.Qt.transpose(1, 2).contiguous().cpu().numpy()
        xi = self.xi.cpu().numpy()
        return [EigenFactorization(lam[i], Q[i], xi[i]) for i in range(len(self.ops))]


def eig_tridiag_device(ops) -> list[EigenFactorization]:
    """Batched ``eig_tridiag`` (operators.py:371-382) of operators that share
    one extent; returns host ``EigenFactorization`` objects in input order."""
    ops = list(ops)
    if not ops:
        return []
    batch = _EigBatch(ops[0].n)
    idx = [batch.add(op) for op in ops]
    if any(op.n != batch.n for op in ops):
        raise ValueError("eig_tridiag_device needs operators of one extent")
    batch.solve().check()
    facs = batch.factorizations()
    return [facs[i] for i in idx]


def _phi1_matrices(batch: _EigBatch, mats, scales):
    """phi1(s_k A_{m_k}) for every (operator index, scale) pair, on device."""
    import torch

    nset, n = len(mats), batch.n
    out = torch.empty((nset, n, n), dtype=torch.float64, device="cuda")
    mat = torch.tensor(mats, dtype=torch.int32, device="cuda")
    s = _dev(scales)
    for lo in range(0, nset, _MAX_SETS):  # one launch takes at most 65535 sets (grid z extent)
        hi = min(nset, lo + _MAX_SETS)
        _native.check(_native.lib().cg_setup_phi1_matrix(hi - lo, n, batch.lam.data_ptr(), batch.Qt.data_ptr(),
                                                         batch.xi.data_ptr(), mat[lo:hi].data_ptr(),
                                                         s[lo:hi].data_ptr(), out[lo:hi].data_ptr(), _stream()),
                      "cg_setup_phi1_matrix")
    return out


def _phi1_outer(f1, f2, f3, scales):
    """phi1(s * f1 (x) f2 [(x) f3]) for every set; factors are [nset][n_i]
    CUDA tensors (f3 may be None)."""
    import torch

    nset, n1, n2 = f1.shape[0], f1.shape[1], f2.shape[1]
    n3 = 1 if f3 is None else f3.shape[1]
    shape = (nset, n1, n2) if f3 is None else (nset, n1, n2, n3)
    out = torch.empty(shape, dtype=torch.float64, device="cuda")
    s = _dev(scales)
    f1, f2 = f1.contiguous(), f2.contiguous()
    f3 = None if f3 is None else f3.contiguous()
    for lo in range(0, nset, _MAX_SETS):
        hi = min(nset, lo + _MAX_SETS)
        _native.check(_native.lib().cg_setup_phi1_outer(hi - lo, n1, n2, n3, f1[lo:hi].data_ptr(), f2[lo:hi].data_ptr(),
                                                        None if f3 is None else f3[lo:hi].data_ptr(),
                                                        s[lo:hi].data_ptr(), out[lo:hi].data_ptr(), _stream()),
                      "cg_setup_phi1_outer")
    return out


def phi1_device(x) -> np.ndarray:
    """Elementwise phi1 (phifun.py:23-37) on the device; NumPy in, NumPy out."""
    import torch

    arr = np.asarray(x, dtype=float)
    flat = _dev(arr.ravel())
    out = torch.empty_like(flat)
    _native.check(_native.lib().cg_setup_phi1(flat.numel(), flat.data_ptr(), out.data_ptr(), _stream()),
                  "cg_setup_phi1")
    return out.cpu().numpy().reshape(arr.shape)


def prepare_device(bases, tau: float) -> list[GeometryOps]:
    """``[prepare(b, tau) for b in bases]`` with the eigenproblems, the dense
    phi1 factors and the Phi tensors evaluated on the GPU in batched launches.
    ``bases`` are ComponentOps (ours or the reference's) of one geometry and
    grid; results agree with the host path to rounding (the eigenvectors may
    differ in sign, which no product of the stepper sees)."""
    import torch

    if tau < 0:
        raise ValueError("tau must be nonnegative")
    bases = list(bases)
    if not bases:
        return []
    g = _geometry_name(bases[0].geometry)
    if g not in ("disk", "sphere", "ball", "cylinder"):
        raise ValueError(f"unknown geometry {g!r}")
    shape = bases[0].shape
    if any(_geometry_name(b.geometry) != g or b.shape != shape for b in bases):
        raise NotImplementedError("prepare_device needs bases of one geometry and grid")
    B = len(bases)
    s = np.array([tau * b.coeff for b in bases], dtype=float)

    # distinct operators per axis -> one eigen-solve launch per axis
    axes = {ax: _EigBatch(getattr(bases[0], ax).n) for ax in ("rho", "phi", "z") if getattr(bases[0], ax) is not None}
    where = {ax: [batch.add(getattr(b, ax)) for b in bases] for ax, batch in axes.items()}
    for batch in axes.values():
        batch.solve()
    # dense phi1 factors of every base, one launch per axis
    p1 = {}
    if "rho" in axes:
        p1["rho"] = _phi1_matrices(axes["rho"], where["rho"], s)
    if "phi" in axes and g == "sphere":
        p1["phi"] = _phi1_matrices(axes["phi"], where["phi"], s)
    if "z" in axes:
        p1["z"] = _phi1_matrices(axes["z"], where["z"], s)
    # host closed forms
    th = [_cached(b.theta, "eig_theta", eig_theta) for b in bases]
    lam_theta = _dev(np.stack([t.lambdas for t in th]))
    d_rho = [_rho_weights(b) for b in bases] if "rho" in axes else None
    d_phi = [_cached(b.phi, "sin2", lambda o: np.sin(o.grid) ** -2.0) for b in bases] if "phi" in axes else None
    ones = lambda n: torch.ones((B, n), dtype=torch.float64, device="cuda")  # noqa: E731
    mix_outer = None
    if g == "disk":
        mix = _phi1_outer(_dev(np.stack(d_rho)), lam_theta, None, s)
    elif g == "sphere":
        mix = _phi1_outer(lam_theta, _dev(np.stack(d_phi)), None, s)
    elif g == "ball":
        lam_phi = axes["phi"].lam[torch.tensor(where["phi"], device="cuda")]
        dr = _dev(np.stack(d_rho))
        mix_outer = _phi1_outer(dr, ones(bases[0].theta.n), lam_phi, s)
        mix = _phi1_outer(dr, lam_theta, _dev(np.stack(d_phi)), s)
    else:
        mix = _phi1_outer(_dev(np.stack(d_rho)), lam_theta, ones(bases[0].z.n), s)
    for batch in axes.values():
        batch.check()

    # hand-over: one download per table family
    host = {k: v.cpu().numpy() for k, v in p1.items()}
    mix_h = mix.cpu().numpy()
    mix_outer_h = None if mix_outer is None else mix_outer.cpu().numpy()
    phi_facs = axes["phi"].factorizations() if "phi" in axes else None
    out = []
    for i, b in enumerate(bases):
        kw: dict = dict(A_theta=_cached(b.theta, "dense", lambda o: o.toarray()), Q_theta=th[i].Q,
                        lam_theta=th[i].lambdas)
        if "rho" in axes:
            kw.update(A_rho=_cached(b.rho, "dense", lambda o: o.toarray()), d_rho=d_rho[i], phi1_rho=host["rho"][i])
        if "phi" in axes:
            kw.update(A_phi=_cached(b.phi, "dense", lambda o: o.toarray()), d_phi=d_phi[i],
                      phi_fac=phi_facs[where["phi"][i]])
            if g == "sphere":
                kw["phi1_phi"] = host["phi"][i]
        if "z" in axes:
            kw.update(A_z=_cached(b.z, "dense", lambda o: o.toarray()), phi1_z=host["z"][i])
        kw["phi_mix"] = PhiTensor(field=mix_h[i], tau_scale=float(s[i]))
        if mix_outer_h is not None:
            kw["phi_mix_outer"] = PhiTensor(field=mix_outer_h[i], tau_scale=float(s[i]))
        out.append(GeometryOps(base=b, tau=tau, **kw))
    return out
