"""The drop-in `tensor` module on the GPU against the reference's own tensor
tests (pkg/tests/test_tensor.py): loop oracle <= 1e-13 (:48-54), identity
bitwise (:40-45), Kronecker duality <= 1e-13 (:57-104), shape errors, plus
BASELINE-sized products against NumPy's contraction."""

import numpy as np
import pytest

from paper_2604_11558_b200 import tensor

pytestmark = pytest.mark.gpu


def loop_mode_product(mu, L, T):
    out = np.zeros_like(np.asarray(T, dtype=float))
    for idx in np.ndindex(*T.shape):
        acc = 0.0
        for m in range(T.shape[mu - 1]):
            src = list(idx)
            src[mu - 1] = m
            acc += L[idx[mu - 1], m] * T[tuple(src)]
        out[idx] = acc
    return out


def test_vec_unvec_roundtrip_and_linearization():
    rng = np.random.RandomState(0)
    for dims in [(5,), (3, 4), (2, 3, 4)]:
        T = rng.randn(*dims)
        assert np.array_equal(tensor.unvec(tensor.vec(T), dims), T)
    T = np.zeros((3, 4, 2))
    T[1, 2, 1] = 7.0
    assert tensor.vec(T)[1 + 2 * 3 + 1 * 3 * 4] == 7.0
    with pytest.raises(ValueError):
        tensor.unvec(np.zeros(5), (2, 3))


@pytest.mark.parametrize("dims", [(4, 3, 5), (6, 8), (7,), (16, 32, 10), (100, 100, 100)])
def test_mode_product_identity_is_bitwise(dims):
    rng = np.random.RandomState(1)
    T = rng.randn(*dims)
    for mu in range(1, len(dims) + 1):
        out = tensor.mode_product(mu, np.eye(dims[mu - 1]), T)
        assert np.array_equal(out, T), (dims, mu)


@pytest.mark.parametrize("dims", [(3, 3, 3), (4, 5), (5,), (3, 4, 6), (7, 2, 5)])
def test_mode_product_matches_loop_oracle(dims):
    rng = np.random.RandomState(2)
    T = rng.randn(*dims)
    for mu in range(1, len(dims) + 1):
        L = rng.randn(dims[mu - 1], dims[mu - 1])
        out = tensor.mode_product(mu, L, T)
        assert out.shape == T.shape
        assert np.max(np.abs(out - loop_mode_product(mu, L, T))) <= 1e-13, (dims, mu)


def test_mode_products_satisfy_the_kronecker_identity():
    """vec(T x1 L1 x2 L2 [x3 L3]) = (L3 kron L2 kron L1) vec(T)."""
    rng = np.random.RandomState(3)
    for dims in [(4, 5), (3, 4, 2)]:
        T = rng.randn(*dims)
        Ls = [rng.randn(n, n) for n in dims]
        out = tensor.tucker(T, Ls)
        K = Ls[0]
        for L in Ls[1:]:
            K = np.kron(L, K)
        assert np.max(np.abs(tensor.vec(out) - K @ tensor.vec(T))) <= 1e-13
        # skipped / None modes are left untouched
        part = tensor.tucker(T, [Ls[0]] + [None] * (len(dims) - 1))
        assert np.max(np.abs(part - np.tensordot(Ls[0], T, axes=([1], [0])))) <= 1e-13
        assert np.array_equal(tensor.tucker(T, Ls, skip=set(range(1, len(dims) + 1))), T)


@pytest.mark.parametrize("dims", [(64, 128), (128, 256), (512, 256), (64, 128, 128), (100, 100, 100), (30, 50, 30)])
def test_baseline_sized_products_match_numpy(dims):
    rng = np.random.RandomState(4)
    T = rng.randn(*dims)
    for mu in range(1, len(dims) + 1):
        n = dims[mu - 1]
        L = rng.randn(n, n) / np.sqrt(n)
        want = np.moveaxis(np.tensordot(L, T, axes=([1], [mu - 1])), 0, mu - 1)
        got = tensor.mode_product(mu, L, T)
        assert np.max(np.abs(got - want)) <= 1e-13 * max(1.0, np.max(np.abs(want))), (dims, mu)


def test_mode_product_accepts_and_returns_device_tensors():
    import torch

    rng = np.random.RandomState(5)
    T = rng.randn(12, 20, 16)
    L = rng.randn(20, 20)
    dev = tensor.mode_product(2, L, torch.from_numpy(T).cuda())
    assert isinstance(dev, torch.Tensor) and dev.is_cuda and dev.shape == (12, 20, 16)
    assert np.max(np.abs(dev.cpu().numpy() - tensor.mode_product(2, L, T))) == 0.0


def test_mode_product_rejects_what_the_reference_rejects():
    T = np.zeros((3, 4))
    with pytest.raises(ValueError):
        tensor.mode_product(3, np.eye(3), T)
    with pytest.raises(ValueError):
        tensor.mode_product(0, np.eye(3), T)
    with pytest.raises(ValueError):
        tensor.mode_product(1, np.eye(4), T)
    with pytest.raises(ValueError):
        tensor.mode_product(2, np.zeros((4, 3)), T)
    with pytest.raises(ValueError):
        tensor.tucker(T, [np.eye(3)])


def test_hadamard_matches_numpy_and_rejects_shape_mismatch():
    rng = np.random.RandomState(6)
    for dims in [(5,), (3, 4), (7, 2, 5), (100, 100, 100)]:
        A, B = rng.randn(*dims), rng.randn(*dims)
        assert np.array_equal(tensor.hadamard(A, B), A * B)
    with pytest.raises(ValueError):
        tensor.hadamard(np.zeros((2, 3)), np.zeros((3, 2)))
