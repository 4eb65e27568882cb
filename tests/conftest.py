import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden.npz")))


@pytest.fixture(scope="session")
def refo():
    """The compiled reference (oracle/_ref) — the parity checker."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    return ref


@pytest.fixture(scope="session")
def A():
    """The device library (fails loudly if it is missing: no CPU fallback)."""
    import paper_2006_15234_b200.api as api
    api.default_context()
    return api


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(params=[1, 2], ids=["overlap_auto", "overlap_forced"])
def faithful(A, request):
    """Reference-faithful orthogonalisation basis (elementwise parity of t1/t2),
    with the eigensolver/operator-application overlap (A (Z P) = (A Z) P on two
    streams) at its default size threshold and forced on every einsumsvd."""
    ctx = A.default_context()
    ctx.set_option("orth_mode", 0)
    ctx.set_option("overlap", request.param)
    yield A
    ctx.set_option("orth_mode", 0)
    ctx.set_option("overlap", 1)


@pytest.fixture
def cholqr(A):
    """CholeskyQR2 orthogonalisation (same spans, other basis)."""
    ctx = A.default_context()
    ctx.set_option("orth_mode", 1)
    yield A
    ctx.set_option("orth_mode", 0)


def mps_fidelity(a, b):
    """|<a|b>| / (||a|| ||b||) for two MPS given as lists of (p, l, r) arrays."""
    def ov(x, y):
        l = np.ones((1, 1), dtype=complex)
        for s, t in zip(x, y):
            l = np.einsum("ab,pac,pbd->cd", l, s.conj(), t)
        return l[0, 0]
    return abs(ov(a, b)) / np.sqrt(abs(ov(a, a)) * abs(ov(b, b)))
