"""The opt-in Hermitian Gram kernel (csrc/gram.cu, option gemm_gram): G = Z^H Z of a tall complex Z from
the upper-triangle DMMA blocks of the interleaved real product, split over rows
with a fixed-order reduction -- against numpy at 1e-13, exactly Hermitian,
deterministic, and equal (to rounding) to the generic complex GEMM route it
replaces (option gemm_gram = 0)."""
import numpy as np
import pytest

from oracle import peps_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture
def gram_on(A):
    ctx = A.default_context()
    ctx.set_option("gemm_gram", 1)
    yield A
    ctx.set_option("gemm_gram", 0)


@pytest.mark.parametrize("rows,k", [(2048, 1), (2048, 3), (5000, 8), (4096, 41), (10007, 64), (262144, 72),
                                    (2049, 72), (70000, 17)])
def test_gram_kernel_matches_numpy(gram_on, rows, k):
    A = gram_on
    z = O.random_tensor((rows, k), rows + k)
    g = A.gram(z).numpy()
    want = z.conj().T @ z
    assert np.linalg.norm(g - want) <= 1e-13 * np.linalg.norm(want)
    assert np.array_equal(g, g.conj().T)  # Hermitian by construction
    assert np.all(np.diag(g).imag == 0.0)
    assert np.array_equal(A.gram(z).numpy(), g)  # deterministic


def test_gram_kernel_vs_generic_gemm_route(gram_on):
    A = gram_on
    ctx = A.default_context()
    z = O.random_tensor((262144 // 4, 8, 72), 3)
    g1 = A.gram(z).numpy()
    ctx.set_option("gemm_gram", 0)
    g0 = A.gram(z).numpy()
    assert np.linalg.norm(g1 - g0) <= 1e-14 * np.linalg.norm(g0)
