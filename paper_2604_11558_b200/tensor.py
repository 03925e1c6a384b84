"""Drop-in for the reference's ``curvipat.tensor`` (tensor.py:1-101): mu-mode
products, the Tucker operator, Hadamard products and vec/unvec, with the
products evaluated on the GPU.

``mode_product(mu, L, field)`` is the reference's one-DGEMM contraction
(``np.tensordot`` + ``moveaxis``, tensor.py:31-49) run as the engine's batched
FP64 DMMA GEMM on a single field: the unfolding of mode ``mu`` is folded into
the TMA tensor maps (``cg_product_create`` / ``cg_product_apply``), nothing is
permuted.  Same names, argument meaning and errors as the reference; NumPy
arrays in give NumPy arrays out, CUDA ``torch`` tensors give CUDA tensors.
Inside the steppers these products never run on their own -- the step kernels
fuse them with their neighbours -- so this module exists for API parity and for
testing the GEMM the way the reference tests its own
(tests/test_tensor.py:40-104).  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict

import numpy as np

from . import _native


def vec(field) -> np.ndarray:
    """Flatten a field with the first index fastest (tensor.py:18-20)."""
    return np.asarray(field).reshape(-1, order="F")


def unvec(w, dims) -> np.ndarray:
    """Inverse of :func:`vec` for the given dims (tensor.py:23-28)."""
    w = np.asarray(w)
    if w.size != int(np.prod(dims)):
        raise ValueError(f"cannot reshape {w.size} values into dims {tuple(dims)}")
    return w.reshape(dims, order="F")


class _Product:
    """One (mode, dims, operator) product handle; freed with the cache entry."""

    def __init__(self, mu: int, dims: tuple[int, ...], L: np.ndarray):
        self._lib = _native.lib()
        arr = (ctypes.c_int * len(dims))(*dims)
        Lc = np.ascontiguousarray(L, dtype=np.float64)
        handle = ctypes.c_void_p()
        _native.check(self._lib.cg_product_create(mu, len(dims), arr, _native.dptr(Lc), ctypes.byref(handle)),
                      "cg_product_create")
        self._h = handle

    def apply(self, T, out):
        import torch

        _native.check(self._lib.cg_product_apply(self._h, T.data_ptr(), out.data_ptr(),
                                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                      "cg_product_apply")

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                import torch

                torch.cuda.synchronize()  # a product may still be running on the handle's operator
                self._lib.cg_product_destroy(self._h)
                self._h = None
        except Exception:
            pass


_CACHE: OrderedDict = OrderedDict()
_CACHE_MAX = 16


def _handle(mu: int, dims: tuple[int, ...], L: np.ndarray) -> _Product:
    key = (mu, dims, L.shape, L.tobytes())
    hit = _CACHE.get(key)
    if hit is None:
        hit = _Product(mu, dims, L)
        _CACHE[key] = hit
        if len(_CACHE) > _CACHE_MAX:
            _CACHE.popitem(last=False)
    else:
        _CACHE.move_to_end(key)
    return hit


def mode_product(mu: int, L, field):
    """Multiply the square matrix L along mode ``mu`` (1-based) of the field:
    ``mode_product(1, L, T)[i, j, k] = sum_m L[i, m] T[m, j, k]`` and
    analogously along the other modes (tensor.py:31-49)."""
    import torch

    on_device = isinstance(field, torch.Tensor)
    L = np.asarray(L.detach().cpu().numpy() if isinstance(L, torch.Tensor) else L, dtype=np.float64)
    shape = tuple(field.shape)
    ndim = len(shape)
    if not 1 <= mu <= ndim:
        raise ValueError(f"mode {mu} out of range for order-{ndim} field")
    axis = mu - 1
    if L.ndim != 2 or L.shape[0] != L.shape[1] or L.shape[1] != shape[axis]:
        raise ValueError(f"matrix of shape {L.shape} does not fit mode {mu} of field with dims {shape}")
    if ndim > 3:
        raise NotImplementedError("fields of order 1, 2 or 3 (as the reference's geometries)")
    if on_device:
        if not field.is_cuda or field.dtype != torch.float64:
            raise ValueError("device fields must be CUDA float64 tensors")
        T = field.contiguous()
    else:
        T = torch.from_numpy(np.ascontiguousarray(np.asarray(field, dtype=np.float64))).cuda()
    # the GEMM wants an order-2/3 field whose contiguous extent is even: an
    # order-1 field becomes a one-column matrix, an odd last extent gets one zero
    # column (and, along that mode, the operator one zero row and column)
    mu_e, dims = mu, list(shape)
    if ndim == 1:
        T = T.reshape(shape[0], 1)
        dims = [shape[0], 1]
    Le = L
    if dims[-1] % 2:
        pad = torch.zeros((*dims[:-1], 1), dtype=torch.float64, device="cuda")
        T = torch.cat([T, pad], dim=-1).contiguous()
        if mu_e == len(dims):
            Le = np.zeros((L.shape[0] + 1, L.shape[0] + 1))
            Le[:-1, :-1] = L
        dims[-1] += 1
    out = torch.empty_like(T)
    _handle(mu_e, tuple(dims), Le).apply(T, out)
    out = out[..., : shape[-1]] if ndim > 1 else out[:, 0]
    out = out.reshape(shape)
    return out.contiguous() if on_device else out.cpu().numpy()


def tucker(field, matrices, skip=None):
    """Concatenated mode products in ascending mode order; ``None`` entries
    and modes listed in ``skip`` are left untouched (tensor.py:52-74)."""
    ndim = len(field.shape)
    if len(matrices) != ndim:
        raise ValueError(f"expected {ndim} mode matrices, got {len(matrices)}")
    skip = skip or set()
    out = field
    for mu, L in enumerate(matrices, start=1):
        if mu in skip or L is None:
            continue
        out = mode_product(mu, L, out)
    return out


def hadamard(A, B):
    """Elementwise product of two fields with identical dims (tensor.py:77-83)."""
    import torch

    if tuple(A.shape) != tuple(B.shape):
        raise ValueError(f"shape mismatch {tuple(A.shape)} vs {tuple(B.shape)}")
    on_device = isinstance(A, torch.Tensor) and isinstance(B, torch.Tensor)

    def dev(x):
        if isinstance(x, torch.Tensor):
            if not x.is_cuda or x.dtype != torch.float64:
                raise ValueError("device fields must be CUDA float64 tensors")
            return x.contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).cuda()

    a, b = dev(A), dev(B)
    out = torch.empty_like(a)
    if a.numel():
        _native.check(_native.lib().cg_hadamard(a.data_ptr(), b.data_ptr(), out.data_ptr(), a.numel(),
                                                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                      "cg_hadamard")
    return out if on_device else out.cpu().numpy()
