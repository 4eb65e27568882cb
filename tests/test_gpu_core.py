"""GPU parity of the einsumsvd building blocks against the reference.

Models: proj/tests/test_decomposition.cpp (implicit operator, Gram
orthogonalisation, randomized SVD, einsumsvd) and test_einsum.cpp /
test_linalg.cpp.  Every call goes through the C ABI (lib/libpeps_b200.so).
Tolerances are the reference tests' own where they exist; parity against the
reference's outputs (golden fixtures / live oracle) is 1e-10 relative unless
stated (bar: 1e-8 on gauge-invariant quantities, north_star).
"""
import numpy as np
import pytest

from conftest import rel
from oracle import peps_oracle as O

pytestmark = pytest.mark.gpu


def test_random_tensor_bitwise(A, golden):
    for i, s in enumerate(golden["rng_seeds"]):
        assert np.array_equal(A.random_tensor((3, 5), int(s)).numpy(), golden["rng_complex"][i])
        assert np.array_equal(A.random_tensor((3, 5), int(s), real=True).numpy(), golden["rng_real"][i])
    big = A.random_tensor((8, 8, 64, 8, 8, 72), 12345).numpy()
    assert np.array_equal(big.reshape(-1)[:4096], O.random_tensor((4096,), 12345))
    assert np.array_equal(big.reshape(-1)[-7:], O.random_tensor((big.size,), 12345)[-7:])


@pytest.mark.parametrize("spec,shapes", [
    ("abc,cd->abd", [(6, 7, 8), (8, 9)]),
    ("abc,acd->bd", [(6, 7, 8), (6, 8, 5)]),
    ("ik,kj->ij", [(70, 300), (300, 90)]),
    ("abc,cba->", [(3, 4, 5), (5, 4, 3)]),
    ("ab,cd->abcd", [(3, 4), (5, 2)]),
    ("bij,bjk->bik", [(4, 5, 6), (4, 6, 7)]),
    ("ijk,jkl,lm->im", [(4, 5, 6), (5, 6, 7), (7, 3)]),
    ("aab,bc->ac", [(3, 3, 4), (4, 5)]),
    ("abc->ca", [(3, 4, 5)]),
])
def test_contract_matches_einsum(A, spec, shapes):
    ts = [O.random_tensor(s, 10 + i) for i, s in enumerate(shapes)]
    got = A.contract(spec, *ts).numpy()
    assert rel(got, np.einsum(spec, *ts)) < 1e-13


def _two_layer(r, m, seed):
    v = O.random_tensor((m, r, r, m, r, r), seed)
    s = O.random_tensor((r, r, m, m), seed + 1)
    b = O.random_tensor((2, r, r, r, r), seed + 2)
    return [v, s, b.conj(), b], ["apqsmn", "uvst", "dumbe", "dvncf"]


def test_implicit_apply_adjoint_materialize(A):
    ts, labs = _two_layer(3, 5, 11)
    op = A.ImplicitOperator(ts, labs, "apq", "bctef")
    ro = O.ImplicitOperator(ts, labs, "apq", "bctef")
    q = O.random_tensor((3, 3, 5, 3, 3, 7), 15)
    p = O.random_tensor((5, 3, 3, 7), 16)
    assert rel(op.apply(q).numpy(), ro.apply(q)) < 1e-13
    assert rel(op.adjoint_apply(p).numpy(), ro.adjoint_apply(p)) < 1e-13
    assert rel(op.materialize().numpy(), ro.materialize()) < 1e-13
    # <P, A Q> == <A* P, Q>   (test_decomposition.cpp:56-67)
    lhs = np.vdot(p, op.apply(q).numpy())
    rhs = np.vdot(op.adjoint_apply(p).numpy(), q)
    assert abs(lhs - rhs) < 1e-11 * abs(lhs)


def test_identity_network(A):
    op = A.ImplicitOperator([np.eye(2, dtype=complex)], ["rc"], "r", "c")
    q = O.random_tensor((2, 1), 4)
    assert np.abs(op.apply(q).numpy() - q).max() < 1e-15


def test_gram_orthogonalize(A, golden):
    q, r = A.gram_orthogonalize(O.random_tensor((64, 4), 17), 1)
    assert rel(q.numpy(), golden["gram_q"]) < 1e-10 and rel(r.numpy(), golden["gram_r"]) < 1e-10
    base = O.random_tensor((32, 3), 23)
    a2 = np.stack([base[:, 0], base[:, 1], base[:, 0], base[:, 2]], axis=1)
    q2, r2 = A.gram_orthogonalize(a2, 1)
    q2, r2 = q2.numpy(), r2.numpy()
    assert np.abs(q2.conj().T @ q2 - np.eye(4)).max() < 1e-6
    assert rel(q2 @ r2, a2) < 1e-5
    # basis column (test_decomposition.cpp:84-92)
    e = np.zeros((8, 1), dtype=complex)
    e[0, 0] = 1
    qb, rb = A.gram_orthogonalize(e, 1)
    assert abs(qb.numpy()[0, 0] - 1) < 1e-12 and abs(rb.numpy()[0, 0] - 1) < 1e-12


def test_gram_zero_operator_raises(A):
    with pytest.raises(A.PepsError, match="NumericalError"):
        A.gram_orthogonalize(np.zeros((8, 2), dtype=complex), 1)


def test_svd_matches_reference(A, refo):
    for shape, split in [((40, 3, 6), 1), ((5, 30), 1), ((4, 4, 4, 4), 2), ((32, 32), 1)]:
        t = O.random_tensor(shape, 21)
        u, s, v = A.svd(t, split)
        ur, sr, vr = refo.svd(t, split)
        assert rel(s, sr) < 1e-13
        assert rel(u.numpy(), ur) < 1e-11 and rel(v.numpy(), vr) < 1e-11


def test_rsvd_exact_rank_diagonal(A, golden):
    d = np.zeros((4, 4), dtype=complex)
    d[0, 0], d[1, 1], d[2, 2] = 3, 2, 1
    t = A.randomized_svd(A.ImplicitOperator([d], ["rc"], "r", "c"), A.TruncationPolicy(3, 1e-14),
                         A.RsvdConfig(2, -1, 7))
    assert len(t.s) == 3 and np.allclose(t.s, [3, 2, 1], atol=1e-10)


def test_rsvd_rank5_recovery(A, golden):
    l, r = O.random_tensor((8, 5), 41), O.random_tensor((5, 8), 42)
    t = A.randomized_svd(A.ImplicitOperator([l @ r], ["rc"], "r", "c"), A.TruncationPolicy(5, 1e-14),
                         A.RsvdConfig(2, -1, 7))
    rec = (t.u.numpy() * t.s) @ t.v.numpy()
    assert rel(rec, l @ r) < 1e-8
    assert rel(t.s, golden["rank5_s"]) < 1e-10


def test_rsvd_deterministic_and_clamped(A):
    a = O.random_tensor((16, 16), 51)
    op = A.ImplicitOperator([a], ["rc"], "r", "c")
    t1 = A.randomized_svd(op, A.TruncationPolicy(6, 1e-14), A.RsvdConfig(2, -1, 99))
    t2 = A.randomized_svd(op, A.TruncationPolicy(6, 1e-14), A.RsvdConfig(2, -1, 99))
    assert np.array_equal(t1.u.numpy(), t2.u.numpy()) and np.array_equal(t1.v.numpy(), t2.v.numpy())
    b = O.random_tensor((4, 6), 71)
    t = A.randomized_svd(A.ImplicitOperator([b], ["rc"], "r", "c"), A.TruncationPolicy(32, 1e-14),
                         A.RsvdConfig(1, -1, 5))
    assert t.rank_clamped and len(t.s) <= 4


def test_rsvd_error_within_optimal_bound(A):
    a = O.random_tensor((32, 32), 61)
    s_full = np.linalg.svd(a, compute_uv=False)
    opt = np.sqrt((s_full[8:] ** 2).sum())
    t = A.randomized_svd(A.ImplicitOperator([a], ["rc"], "r", "c"), A.TruncationPolicy(8, 1e-14),
                         A.RsvdConfig(2, -1, 7))
    err = np.linalg.norm((t.u.numpy() * t.s) @ t.v.numpy() - a)
    assert err <= 1.25 * opt


@pytest.mark.parametrize("absorb", ["split", "left", "right"])
def test_einsumsvd_two_layer_gauge_invariant_cholqr(cholqr, golden, absorb):
    """CholeskyQR2 orthogonalisation: same spans as the reference, so singular
    values, ranks and the product t1 t2 agree (north_star bar)."""
    A = cholqr
    ts, labs = _two_layer(3, 6, 100)
    res = A.einsumsvd(A.ImplicitOperator(ts, labs, "apq", "bctef"), A.TruncationPolicy(6, 1e-14),
                      A.SvdStrategy.implicit_rsvd, A.Absorb[absorb], A.RsvdConfig(2, -1, 11))
    assert res.s.shape == golden[f"es_tl_{absorb}_s"].shape
    assert rel(res.s, golden[f"es_tl_{absorb}_s"]) < 1e-10
    g1, g2 = golden[f"es_tl_{absorb}_t1"], golden[f"es_tl_{absorb}_t2"]
    k = len(res.s)
    prod = res.t1.numpy().reshape(-1, k) @ res.t2.numpy().reshape(k, -1)
    assert rel(prod, g1.reshape(-1, k) @ g2.reshape(k, -1)) < 1e-9


@pytest.mark.parametrize("absorb", ["split", "left", "right"])
def test_einsumsvd_two_layer_matches_reference(faithful, golden, absorb):
    A = faithful
    ts, labs = _two_layer(3, 6, 100)
    res = A.einsumsvd(A.ImplicitOperator(ts, labs, "apq", "bctef"), A.TruncationPolicy(6, 1e-14),
                      A.SvdStrategy.implicit_rsvd, A.Absorb[absorb], A.RsvdConfig(2, -1, 11))
    assert res.s.shape == golden[f"es_tl_{absorb}_s"].shape  # bit-exact rank metadata
    assert rel(res.s, golden[f"es_tl_{absorb}_s"]) < 1e-12
    assert res.t1.shape == golden[f"es_tl_{absorb}_t1"].shape
    assert rel(res.t1.numpy(), golden[f"es_tl_{absorb}_t1"]) < 1e-9
    assert rel(res.t2.numpy(), golden[f"es_tl_{absorb}_t2"]) < 1e-9


def test_einsumsvd_exact_and_chain(faithful, golden):
    A = faithful
    ts, labs = _two_layer(3, 6, 100)
    ex = A.einsumsvd(A.ImplicitOperator(ts, labs, "apq", "bctef"), A.TruncationPolicy(6, 1e-14),
                     A.SvdStrategy.exact)
    assert rel(ex.s, golden["es_tl_exact_s"]) < 1e-12
    chain = [O.random_tensor(s, sd) for s, sd in (((2, 3), 81), ((3, 2, 4), 82), ((4, 5), 83),
                                                    ((5, 3, 2), 84), ((2, 3), 85))]
    op = A.ImplicitOperator(chain, ["ab", "bcd", "de", "efg", "gh"], "ac", "fh")
    want = O.ImplicitOperator(chain, ["ab", "bcd", "de", "efg", "gh"], "ac", "fh").materialize().reshape(4, 9)
    e = A.einsumsvd(op, A.TruncationPolicy(4, 1e-14), A.SvdStrategy.exact)
    i = A.einsumsvd(op, A.TruncationPolicy(4, 1e-14), A.SvdStrategy.implicit_rsvd, A.Absorb.split,
                    A.RsvdConfig(2, -1, 3))
    assert rel(e.t1.numpy().reshape(4, -1) @ e.t2.numpy().reshape(-1, 9), want) < 1e-10
    assert rel(i.t1.numpy().reshape(4, -1) @ i.t2.numpy().reshape(-1, 9), want) < 1e-8
    assert rel(e.s, golden["es_chain_exact_s"]) < 1e-12
    assert rel(i.s, golden["es_chain_rsvd_s"]) < 1e-10


def test_absorb_isometries(A):
    a = O.random_tensor((4, 4), 3)
    op = A.ImplicitOperator([a], ["rc"], "r", "c")
    left = A.einsumsvd(op, A.TruncationPolicy(4, 1e-14), A.SvdStrategy.exact, A.Absorb.left)
    right = A.einsumsvd(op, A.TruncationPolicy(4, 1e-14), A.SvdStrategy.exact, A.Absorb.right)
    r1 = right.t1.numpy()
    l2 = left.t2.numpy()
    assert np.abs(r1.conj().T @ r1 - np.eye(4)).max() < 1e-12
    assert np.abs(l2 @ l2.conj().T - np.eye(4)).max() < 1e-12
    assert np.abs(left.t1.numpy() @ l2 - r1 @ right.t2.numpy()).max() < 1e-12


def test_bond_cap_and_finiteness(A):
    for seed in range(4):
        a = O.random_tensor((4, 5, 3), 900 + seed)
        b = O.random_tensor((3, 4, 5), 950 + seed)
        op = A.ImplicitOperator([a, b], ["abm", "mcd"], "ab", "cd")
        for m in (1, 2, 7):
            for strat in (A.SvdStrategy.exact, A.SvdStrategy.implicit_rsvd):
                r = A.einsumsvd(op, A.TruncationPolicy(m, 1e-14), strat, A.Absorb.split, A.RsvdConfig(1, -1, seed))
                k = r.t1.shape[-1]
                assert 1 <= k <= m
                assert np.isfinite(r.t1.numpy()).all() and np.isfinite(r.t2.numpy()).all()


@pytest.mark.parametrize("mode", [0, 1])
def test_einsumsvd_vs_live_reference_larger(A, refo, mode):
    """m=16 r=4 two-layer column: ranks bit-exact, singular values to 1e-10;
    faithful mode also matches t1/t2 elementwise, CholeskyQR2 mode the product."""
    ts, labs = _two_layer(4, 16, 300)
    ctx = A.default_context()
    ctx.set_option("orth_mode", mode)
    try:
        for absorb in ("left", "right"):
            res = A.einsumsvd(A.ImplicitOperator(ts, labs, "apq", "bctef"), A.TruncationPolicy(16, 1e-14),
                              A.SvdStrategy.implicit_rsvd, A.Absorb[absorb], A.RsvdConfig(2, 8, 17))
            want = refo.einsumsvd(ts, labs, "apq", "bctef", 16, 1e-14, "implicit_rsvd", absorb, 2, 8, 17)
            assert res.s.shape == want["s"].shape
            assert rel(res.s, want["s"]) < 1e-10
            k = len(res.s)
            t1, t2 = res.t1.numpy(), res.t2.numpy()
            if mode == 0:
                assert rel(t1, want["t1"]) < 1e-8
                assert rel(t2, want["t2"]) < 1e-8
            assert rel(t1.reshape(-1, k) @ t2.reshape(k, -1),
                       want["t1"].reshape(-1, k) @ want["t2"].reshape(k, -1)) < 1e-9
    finally:
        ctx.set_option("orth_mode", 0)


def test_rank_deficient_probe_falls_back_to_faithful(A, refo):
    """Exact-rank operator with more probes than rank: CholeskyQR breaks down,
    the decomposition is redone on the reference's clamp+completion route."""
    l, r = O.random_tensor((12, 3), 1), O.random_tensor((3, 12), 2)
    a = l @ r
    for mode in (1, 0):
        A.default_context().set_option("orth_mode", mode)
        t = A.randomized_svd(A.ImplicitOperator([a], ["rc"], "r", "c"), A.TruncationPolicy(6, 1e-14),
                             A.RsvdConfig(2, -1, 3))
        want = refo.randomized_svd([a], ["rc"], "r", "c", 6, 1e-14, 2, -1, 3)
        assert t.s.shape == want["s"].shape  # rank metadata: 3 retained of target 6
        assert rel(t.s, want["s"]) < 1e-10
        assert rel((t.u.numpy() * t.s) @ t.v.numpy(), a) < 1e-10
    A.default_context().set_option("orth_mode", 0)


def test_errors_mirror_reference(A):
    with pytest.raises(A.PepsError, match="ShapeError"):
        A.ImplicitOperator([np.eye(2, dtype=complex)], ["rcx"], "r", "c").materialize()
    with pytest.raises(A.PepsError, match="ShapeError"):
        A.contract("ab,bc->ad", np.eye(2, dtype=complex), np.eye(2, dtype=complex))
    with pytest.raises(A.PepsError, match="ValidationError"):
        A.randomized_svd(A.ImplicitOperator([np.eye(2, dtype=complex)], ["rc"], "r", "c"),
                         A.TruncationPolicy(0, 1e-14))


@pytest.mark.parametrize("algo,ws", [(0, 0), (1, 0), (2, 0), (1, 1), (2, 1), (1, 2), (2, 2)],
                         ids=["4m_embed", "3m", "4m_cfrag", "3m_ws", "4m_cfrag_ws", "3m_tma", "4m_cfrag_tma"])
def test_gemm_kernels_all_layouts(A, algo, ws):
    """Every complex GEMM kernel (real embedding, 3M/Gauss, 4M complex
    fragments; classic and persistent warp-specialised bulk-copy variants) on
    every tile configuration (64/72-wide, transposed problems, ragged edges,
    split-K) and operand layout, against numpy at rounding level."""
    ctx = A.default_context()
    ctx.set_option("gemm_algo", algo)
    ctx.set_option("gemm_ws", ws)
    ctx.set_option("gemm_small", 0)  # the tiled kernels on the tiny shapes too
    try:
        shapes = [(70, 90, 300), (64, 64, 64), (72, 72, 72), (128, 300, 64), (65, 70, 17), (5, 7, 3),
                  (200, 72, 130), (72, 200, 33), (64, 72, 64), (72, 64, 48), (33, 65, 129), (1, 1, 1),
                  (8, 300, 256), (300, 8, 256), (72, 72, 5000)]
        for (m, n, k) in shapes:
            for sp in ["ik,kj->ij", "ki,kj->ij", "ik,jk->ij", "ki,jk->ij"]:
                a = O.random_tensor((m, k) if sp[:2] == "ik" else (k, m), m * 7 + k)
                b = O.random_tensor((k, n) if sp[3:5] == "kj" else (n, k), n * 5 + k)
                got = A.contract(sp, a, b).numpy()
                ref = np.einsum(sp, a, b)
                assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (algo, sp, m, n, k)
            # conjugated operand (the adjoint applies of the implicit operator)
            a = O.random_tensor((m, k), m + k)
            b = O.random_tensor((k, n), n + k)
            got = A.contract("ik,kj->ij", a.conj(), b).numpy()
            assert np.abs(got - a.conj() @ b).max() <= 1e-12 * np.abs(a.conj() @ b).max()
    finally:
        ctx.set_option("gemm_algo", 1)
        ctx.set_option("gemm_ws", 0)
        ctx.set_option("gemm_small", 1)


@pytest.mark.parametrize("algo,ws", [(1, 1), (2, 1), (1, 2), (2, 2)], ids=["3m_ws", "4m_ws", "3m_tma", "4m_tma"])
def test_gemm_ws_persistent_tiles_and_batches(A, algo, ws):
    """Persistent warp-specialised GEMM: several tiles per CTA (the producer
    runs ahead across tile boundaries and reuses the offset tables), K tails,
    batched contractions and scattered (permuted) outputs, against numpy."""
    ctx = A.default_context()
    ctx.set_option("gemm_algo", algo)
    ctx.set_option("gemm_ws", ws)
    try:
        for (m, n, k) in [(128, 9000, 64), (64, 20000, 40), (200, 3000, 37), (96, 4100, 128)]:
            a = O.random_tensor((m, k), m + 3 * k)
            b = O.random_tensor((k, n), n + 5 * k)
            ref = a @ b
            got = A.contract("ik,kj->ij", a, b).numpy()
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (algo, m, n, k)
            got = A.contract("ik,kj->ji", a.conj(), b).numpy()
            ref = (a.conj() @ b).T
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (algo, m, n, k)
        a = O.random_tensor((3, 70, 40), 91)
        b = O.random_tensor((3, 40, 2100), 92)
        got = A.contract("bik,bkj->ibj", a, b).numpy()
        ref = np.einsum("bik,bkj->ibj", a, b)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
        # split into output axes (mixed-radix scatter of the epilogue)
        a = O.random_tensor((8, 8, 24), 93)
        b = O.random_tensor((24, 40, 50), 94)
        got = A.contract("pqk,kst->sqtp", a, b).numpy()
        ref = np.einsum("pqk,kst->sqtp", a, b)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    finally:
        ctx.set_option("gemm_algo", 1)
        ctx.set_option("gemm_ws", 0)


def test_gemm_complex_by_real_operands(A):
    """Operands whose imaginary parts are exactly zero (checked on upload) run
    the complex x real kernel (2 real MACs per complex MAC): real x complex,
    complex x real (transposed onto the real-first kernel), real x real,
    conjugated complex operand, ragged edges, split-K, batched, scattered
    output; against numpy at rounding level."""
    ctx = A.default_context()
    rng = np.random.default_rng(5)

    def real(shape):
        return rng.standard_normal(shape).astype(np.complex128)

    ctx.set_option("gemm_small", 0)
    try:
        for (m, n, k) in [(128, 9000, 64), (64, 7000, 128), (70, 90, 300), (5, 7, 3), (64, 64, 64), (100, 300, 4000)]:
            ar, bc = real((m, k)), O.random_tensor((k, n), m + n)
            for spec, a, b in [("ik,kj->ij", ar, bc), ("ik,kj->ji", ar, bc), ("ik,kj->ij", O.random_tensor((m, k), 3), real((k, n))),
                               ("ik,kj->ij", ar, real((k, n))), ("ki,kj->ij", ar.T.copy(), bc), ("ik,jk->ij", ar, bc.T.copy())]:
                ref = np.einsum(spec, a, b)
                got = A.contract(spec, a, b).numpy()
                assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (spec, m, n, k)
            got = A.contract("ik,kj->ij", ar, A.to_device(bc).conj()).numpy()
            ref = ar @ bc.conj()
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
        a = real((3, 70, 40))
        b = O.random_tensor((3, 40, 2100), 92)
        got = A.contract("bik,bkj->ibj", a, b).numpy()
        ref = np.einsum("bik,bkj->ibj", a, b)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    finally:
        ctx.set_option("gemm_real", 1)
        ctx.set_option("gemm_small", 1)


def test_gemm_small_problem_kernel(A):
    """Problems of at most 2^13 complex MACs (K <= 128) run the CUDA-core FMA
    kernel: every operand layout, conjugation, batched and scattered outputs,
    scalars and matrix-vector products, against numpy at rounding level."""
    ctx = A.default_context()
    ctx.set_option("gemm_small", 1)
    for (m, n, k) in [(1, 1, 1), (4, 16, 4), (5, 7, 3), (8, 128, 4), (8, 8, 64), (4, 16, 128), (1, 300, 7), (72, 5, 20)]:
        for sp in ["ik,kj->ij", "ki,kj->ij", "ik,jk->ij", "ki,jk->ij", "ik,kj->ji"]:
            a = O.random_tensor((m, k) if sp[:2] == "ik" else (k, m), m * 7 + k)
            b = O.random_tensor((k, n) if sp[3:5] == "kj" else (n, k), n * 5 + k)
            got = A.contract(sp, a, b).numpy()
            ref = np.einsum(sp, a, b)
            assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max(), (sp, m, n, k)
        a = O.random_tensor((m, k), m + k)
        b = O.random_tensor((k, n), n + k)
        got = A.contract("ik,kj->ij", A.to_device(a).conj(), A.to_device(b).conj()).numpy()
        ref = a.conj() @ b.conj()
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    a = O.random_tensor((3, 7, 4, 5), 91)
    b = O.random_tensor((5, 3, 6, 2), 92)
    got = A.contract("bipk,kbqj->qjbpi", a, b).numpy()
    ref = np.einsum("bipk,kbqj->qjbpi", a, b)
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    ref = np.einsum("ab,b->a", a[0, :, 0, :4], b[0, 0, :4, 0])
    got = A.contract("ab,b->a", a[0, :, 0, :4].copy(), b[0, 0, :4, 0].copy()).numpy()
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
