"""CPU: the numpy restatement (oracle/peps_oracle.py) pinned against the reference's
own outputs (tests/golden, generated from oracle/_ref) and closed-form KATs
from the reference tests."""
import numpy as np
import pytest

from oracle import peps_oracle as O
from paper_2006_15234_b200 import inputs as I
from conftest import rel


def test_splitmix_random_tensor_bitwise(golden):
    for i, s in enumerate(golden["rng_seeds"]):
        assert np.array_equal(O.random_tensor((3, 5), int(s)), golden["rng_complex"][i])
        assert np.array_equal(O.random_tensor_real((3, 5), int(s)), golden["rng_real"][i])
        assert O.derive_seed(int(s), 0x20, 3, 4) == int(golden["rng_derived"][i])
        # the harness generator uses the same stream
        assert I.derive_seed(int(s), 0x20, 3, 4) == int(golden["rng_derived"][i])


def test_gram_orthogonalize_matches_reference(golden):
    a = O.random_tensor((64, 4), 17)
    q, r = O.gram_orthogonalize(a, 1)
    assert rel(q, golden["gram_q"]) < 1e-12 and rel(r, golden["gram_r"]) < 1e-12
    base = O.random_tensor((32, 3), 23)
    a2 = np.stack([base[:, 0], base[:, 1], base[:, 0], base[:, 2]], axis=1)
    q2, r2 = O.gram_orthogonalize(a2, 1)
    assert np.abs(q2.conj().T @ q2 - np.eye(4)).max() < 1e-6  # test_decomposition.cpp:102-117
    assert rel(q2 @ r2, a2) < 1e-5
    with pytest.raises(ArithmeticError):
        O.gram_orthogonalize(np.zeros((8, 2), dtype=complex), 1)


def test_rsvd_kats(golden):
    d = np.zeros((4, 4), dtype=complex)
    d[0, 0], d[1, 1], d[2, 2] = 3, 2, 1
    _, s, _, _ = O.randomized_svd(O.ImplicitOperator([d], ["rc"], "r", "c"), 3, 1e-14, 2, -1, 7)
    assert np.allclose(s, [3, 2, 1], atol=1e-10)  # test_decomposition.cpp:134-145
    assert np.allclose(s, golden["diag321_s"], rtol=1e-12)
    l, r = O.random_tensor((8, 5), 41), O.random_tensor((5, 8), 42)
    u, s, v, _ = O.randomized_svd(O.ImplicitOperator([l @ r], ["rc"], "r", "c"), 5, 1e-14, 2, -1, 7)
    assert rel((u * s) @ v, l @ r) < 1e-8
    assert rel(s, golden["rank5_s"]) < 1e-12


def test_einsumsvd_two_layer_network_matches_reference(golden):
    v = O.random_tensor((6, 3, 3, 6, 3, 3), 100)
    s = O.random_tensor((3, 3, 6, 6), 101)
    b = O.random_tensor((2, 3, 3, 3, 3), 102)
    op = O.ImplicitOperator([v, s, b.conj(), b], ["apqsmn", "uvst", "dumbe", "dvncf"], "apq", "bctef")
    for absorb in ("split", "left", "right"):
        t1, t2, sv, _ = O.einsumsvd(op, 6, 1e-14, "implicit_rsvd", absorb, 2, -1, 11)
        assert rel(sv, golden[f"es_tl_{absorb}_s"]) < 1e-12
        assert rel(t1, golden[f"es_tl_{absorb}_t1"]) < 1e-9
        assert rel(t2, golden[f"es_tl_{absorb}_t2"]) < 1e-9


def test_config1_norm_matches_reference(golden):
    c = I.config1()
    v = O.contract_two_layer(c["sites"], 4, 4, 4, c["seed"], 1, 4)
    assert abs(v - golden["cfg1_norm"][0]) / abs(golden["cfg1_norm"][0]) < 1e-12
    ex = O.inner_exact(c["sites"], 4, 4)
    assert abs(ex - golden["cfg1_exact"][0]) / abs(ex) < 1e-12


def test_row_absorb_matches_reference(golden):
    sites = I.random_peps(3, 5, 3, 71)
    top, phys = I.random_boundary(5, (3, 3), 9, 72)
    out, _ = O.two_layer_apply_row(top, phys, sites, 3, 5, 1, 9, 5, 2, -1, True, 0x20)
    for i, s in enumerate(out):
        assert s.shape == golden[f"row_site{i}"].shape
        assert rel(s, golden[f"row_site{i}"]) < 1e-9


def test_oracle_restatement_vs_live_reference(refo):
    """Restatement vs the compiled reference on a fresh seeded case."""
    c = dict(sites=I.random_peps(5, 5, 2, 5))
    a = O.contract_two_layer(c["sites"], 5, 5, 6, 9, 2, -1)
    b, _ = refo.contract_two_layer(c["sites"], 5, 5, 6, 9, 2, -1)
    assert abs(a - b) / abs(b) < 1e-10


def test_reference_one_layer_families_consistent(refo):
    """The compiled reference's one-layer families agree when the boundary bond
    is not truncated (pins the harness entry used by the GPU parity tests)."""
    from oracle import peps_oracle as O
    g = [O.random_tensor((1 if r == 0 else 2, 1 if c == 0 else 2, 1 if r == 2 else 2, 1 if c == 2 else 2),
                         O.derive_seed(9, r, c)) for r in range(3) for c in range(3)]
    ex = refo.contract_one_layer(g, 3, 3, 0)
    for fam in (1, 2):
        v = refo.contract_one_layer(g, 3, 3, fam, 16, 1)
        assert abs(v - ex) <= 1e-10 * abs(ex)


def test_reference_peps_container_round_trip(refo, tmp_path):
    """save_peps / load_peps of the compiled reference (state.cpp:240-299)."""
    from paper_2006_15234_b200 import inputs as I
    sites = I.random_peps(3, 2, 2, 4)
    refo.save_peps(sites, 3, 2, tmp_path / "s.peps")
    back, rows, cols, d = refo.load_peps(tmp_path / "s.peps")
    assert (rows, cols, d) == (3, 2, 2)
    assert all(np.array_equal(a, b) for a, b in zip(sites, back))


def _classical_tfim_energy(bits, rows, cols, J):
    z = [1 - 2 * b for b in bits]
    e = sum(-J * z[r * cols + c] * z[r * cols + c + 1] for r in range(rows) for c in range(cols - 1))
    return e + sum(-J * z[r * cols + c] * z[(r + 1) * cols + c] for r in range(rows - 1) for c in range(cols))


def test_reference_vqe_ansatz_known_answers(refo):
    """vqe_ansatz_state (drivers.cpp:100-131) pinned by closed forms: zero
    layers is |0...0>; one layer at theta = pi flips every site (Ry(pi)|0> =
    |1>) and the CNOT cascade (horizontal row-major, then vertical) maps the
    basis state classically.  Basis states have <X> = 0, so the TFIM energy
    (H = -J sum ZZ - h sum X) is the classical ZZ sum."""
    rows, cols, J, h = 2, 3, 1.0, 0.5
    _, e0 = refo.vqe_ansatz(rows, cols, 0, [], 2, J, h, 8, 1, 3)
    assert abs(e0 - _classical_tfim_energy([0] * 6, rows, cols, J)) < 1e-12
    bits = [1] * (rows * cols)
    for r in range(rows):
        for c in range(cols - 1):
            bits[r * cols + c + 1] ^= bits[r * cols + c]
    for r in range(rows - 1):
        for c in range(cols):
            bits[(r + 1) * cols + c] ^= bits[r * cols + c]
    sites, e1 = refo.vqe_ansatz(rows, cols, 1, [np.pi] * (rows * cols), 2, J, h, 8, 1, 3)
    assert len(sites) == rows * cols
    assert abs(e1 - _classical_tfim_energy(bits, rows, cols, J)) < 1e-12


def test_fullsize_goldens_are_packaged():
    """The reference-generated full-size goldens the GPU parity tests read
    (tests/golden/make_golden_fullsize.py; hours of reference CPU time) are in the
    tree with the fields those tests use."""
    import os

    import numpy as np

    gdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    want = {"cfg2_col": ["s"], "cfg2_row": ["bb", "xb", "shapes"], "cfg3": ["norm", "z", "terms"],
            "cfg3_pert": ["norm", "z"], "cfg5_8x8": ["norm", "values", "terms"],
            "cfg5_8x8_pert": ["norm", "values"], "cfg5_12x12_norm": ["norm"], "cfg5_12x12_norm_pert": ["norm"]}
    for name, keys in want.items():
        g = np.load(os.path.join(gdir, f"fullsize_{name}.npz"))
        for k in keys:
            assert k in g.files, (name, k)
    g5 = np.load(os.path.join(gdir, "fullsize_cfg5_8x8.npz"))
    assert g5["values"].shape == (57,) and g5["terms"].shape == (57, 5)
