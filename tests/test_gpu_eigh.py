"""GPU Hermitian eigensolver (the k x k kernel under Gram orthogonalisation).

Models proj/tests/test_linalg.cpp:166-190 (descending order, Pauli X,
reconstruction of a random Hermitian matrix) and extends it with the spectra the
divide-and-conquer deflation paths see: exact multiplicities, graded and
clustered eigenvalues, diagonal and zero matrices, Wilkinson-type close pairs,
sketch Gram matrices at large scale.  Both solvers (divide and conquer, Jacobi)
run every case.  Bars: residual ||A X - X L|| and orthogonality ||X^H X - I||
at a few n eps ||A||; eigenvalues against LAPACK at n eps ||A||; phase-fixed
vectors against the reference's eigh where the spectrum is well separated.
"""
import numpy as np
import pytest

from oracle import peps_oracle as O

pytestmark = pytest.mark.gpu

EPS = 2.220446049250313e-16


def _herm(n, seed):
    a = O.random_tensor((n, n), seed)
    return 0.5 * (a + a.conj().T)


def _with_spectrum(w, seed):
    n = len(w)
    q, _ = np.linalg.qr(O.random_tensor((n, n), seed))
    return (q * np.asarray(w, dtype=float)) @ q.conj().T


def _cases():
    rng = np.random.default_rng(7)
    cases = {}
    for n in (1, 2, 3, 5, 16, 31, 32, 33, 64, 72, 100, 129, 256):
        cases[f"random{n}"] = _herm(n, 100 + n)
    cases["graded72"] = _with_spectrum(np.logspace(0, -15, 72), 3)
    cases["mult72"] = _with_spectrum([1.0] * 30 + [0.5] * 30 + list(np.linspace(2, 3, 12)), 4)
    cases["identity40"] = np.eye(40, dtype=complex)
    cases["zero8"] = np.zeros((8, 8), dtype=complex)
    cases["diag50"] = np.diag(rng.standard_normal(50)).astype(complex)
    cases["cluster64"] = _with_spectrum(1.0 + 1e-12 * rng.standard_normal(64), 5)
    w21 = np.diag(np.abs(np.arange(-10, 11)).astype(float)) + np.diag(np.ones(20), 1) + np.diag(np.ones(20), -1)
    cases["wilkinson21"] = w21.astype(complex)
    y = O.random_tensor((4096, 72), 9) * 1e20
    cases["sketch_gram72"] = y.conj().T @ y
    cases["negdef20"] = -_with_spectrum(np.linspace(1, 2, 20), 6)
    tri = np.diag(rng.standard_normal(48)) + np.diag(1e-17 * np.ones(47), 1) + np.diag(1e-17 * np.ones(47), -1)
    cases["tiny_coupling48"] = tri.astype(complex)
    return cases


CASES = _cases()


@pytest.fixture(params=[0, 1, 2], ids=["auto", "jacobi", "dc"])
def solver(A, request):
    ctx = A.default_context()
    ctx.set_option("eig_solver", request.param)
    yield request.param
    ctx.set_option("eig_solver", 0)


@pytest.mark.parametrize("name", sorted(CASES))
def test_eigh_residual_orthogonality(A, solver, name):
    m = CASES[name]
    n = m.shape[0]
    w, v = A.eigh(m)
    x = v.numpy()
    norm = max(np.linalg.norm(m), 1e-300)  # Frobenius: Jacobi leaves off-diagonals < n eps ||A||_F
    assert np.all(np.diff(w) <= 0), "descending order"
    ref = np.linalg.eigvalsh(0.5 * (m + m.conj().T))[::-1]
    assert np.abs(w - ref).max() <= 8 * n * EPS * norm + 1e-300
    if np.abs(m).max() > 0:
        assert np.abs(m @ x - x * w).max() <= 8 * n * EPS * norm
    assert np.abs(x.conj().T @ x - np.eye(n)).max() <= 8 * n * EPS + 1e-14


@pytest.mark.parametrize("name", ["random5", "random33", "random72", "random129", "negdef20", "sketch_gram72"])
def test_eigh_matches_reference_vectors(A, solver, name):
    m = CASES[name]
    wr, xr = O.eigh(m)
    w, v = A.eigh(m)
    x = v.numpy()
    gap = np.min(np.abs(np.diff(wr))) / np.abs(wr).max()
    assert gap > 1e-6
    # eigenvector error ~ eps / relative gap
    assert np.abs(x - xr).max() <= 1e3 * m.shape[0] * EPS / gap


def test_eigh_reference_cases(A, solver):
    w, v = A.eigh(np.diag([1.0, 2.0]).astype(complex))  # test_linalg.cpp:166
    assert np.allclose(w, [2.0, 1.0], rtol=0, atol=1e-15)
    w, v = A.eigh(np.array([[0, 1], [1, 0]], dtype=complex))  # Pauli X
    assert np.allclose(w, [1.0, -1.0], rtol=0, atol=1e-15)


def test_eigh_rejects_non_hermitian(A, solver):
    from paper_2006_15234_b200._lib import PepsError
    m = O.random_tensor((6, 6), 3)
    with pytest.raises(PepsError):
        A.eigh(m)


@pytest.mark.parametrize("solver", [0, 1, 2], ids=["auto", "jacobi", "dc"])
def test_eigh_scale_invariant_extreme_magnitudes(A, solver):
    """Gram matrices of unnormalised states reach |G| ~ 1e171 (8x8 TFIM after
    100 ITE steps); squares of such entries overflow.  The solver scales by an
    exact power of two: eigenvectors are bitwise those of the unscaled matrix
    and eigenvalues scale exactly, for 2^+560 and 2^-500."""
    ctx = A.default_context()
    ctx.set_option("eig_solver", solver)
    try:
        m = _herm(72, 5) @ _herm(72, 6)
        m = m @ m.conj().T  # positive definite Gram-like
        w0, v0 = A.eigh(m)
        for e in (560, -500):
            w, v = A.eigh(m * 2.0 ** e)
            assert np.array_equal(v.numpy(), v0.numpy())
            assert np.array_equal(np.asarray(w), np.asarray(w0) * 2.0 ** e)
    finally:
        ctx.set_option("eig_solver", 0)
