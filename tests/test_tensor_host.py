"""Host-side pieces of the drop-in tensor module (no GPU): vec / unvec keep the
reference's first-index-fastest convention (tensor.py:18-28,
tests/test_tensor.py:20-37) and the argument checks of mode_product / tucker /
hadamard raise before any device work (tensor.py:40-46, :63-66, :80-82)."""

import numpy as np
import pytest

from paper_2604_11558_b200 import tensor


def test_vec_unvec_roundtrip_bitwise():
    rng = np.random.RandomState(0)
    for dims in [(5,), (3, 4), (2, 3, 4)]:
        T = rng.randn(*dims)
        assert np.array_equal(tensor.unvec(tensor.vec(T), dims), T)


def test_vec_linearization_first_index_fastest():
    T = np.zeros((3, 4, 2))
    T[1, 2, 1] = 7.0
    assert tensor.vec(T)[1 + 2 * 3 + 1 * 3 * 4] == 7.0


def test_unvec_rejects_bad_size():
    with pytest.raises(ValueError):
        tensor.unvec(np.zeros(5), (2, 3))


def test_argument_errors_are_raised_on_the_host():
    T = np.zeros((3, 4))
    for mu, L in [(3, np.eye(3)), (0, np.eye(3)), (1, np.eye(4)), (2, np.zeros((4, 3)))]:
        with pytest.raises(ValueError):
            tensor.mode_product(mu, L, T)
    with pytest.raises(ValueError):
        tensor.tucker(T, [np.eye(3)])
    with pytest.raises(ValueError):
        tensor.hadamard(np.zeros((2, 3)), np.zeros((3, 2)))
