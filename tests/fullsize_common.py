"""Shared definitions of the full-size parity cases (test infrastructure).

Used by tests/golden/make_golden_fullsize.py (which runs the reference) and by
tests/test_gpu_fullsize.py (which runs the device library), so both sides see
exactly the same seeded inputs and the same gauge-invariant observables.
"""
from __future__ import annotations

import numpy as np

from paper_2006_15234_b200 import inputs as I

CFG2_COL_SEED = 42


def cfg2_column_net(seed=CFG2_COL_SEED):
    """One interior column of the config-2 row absorb (contraction.cpp:293-299):
    pending v (a,p,q,s,m,n) = (64,8,8,64,8,8), top site (8,8,64,64), bra/ket
    (2,8,8,8,8), N(0,1) entries; sketch seed derive_seed(seed, 0x20, 1, 3)."""
    v = I.gaussian((64, 8, 8, 64, 8, 8), seed)
    s = I.gaussian((8, 8, 64, 64), seed + 1)
    b = I.gaussian((2, 8, 8, 8, 8), seed + 2)
    return [v, s, b.conj(), b], ["apqsmn", "uvst", "dumbe", "dvncf"], I.derive_seed(seed, 0x20, 1, 3)


def probe_mps(shapes, seed=99):
    """A fixed seeded MPS with the given (p, l, r) site shapes."""
    return [I.gaussian(tuple(int(e) for e in sh), I.derive_seed(seed, c)) for c, sh in enumerate(shapes)]


def chain_overlap(x, y):
    """<x|y> of two MPS with sites (p, l, r): the full contraction over every
    physical index, invariant under any gauge transformation on the bonds."""
    env = np.ones((1, 1), dtype=np.complex128)
    for a, b in zip(x, y):
        env = np.einsum("ab,pac,pbd->cd", env, a.conj(), b, optimize=True)
    return complex(env[0, 0])


def boundary_overlaps(sites):
    """(<b|b>, <x|b>) for an emitted two-layer boundary b (sites (pb*pk, l, r))."""
    x = probe_mps([s.shape for s in sites])
    return chain_overlap(sites, sites), chain_overlap(x, sites)


def cfg5_small(n=8):
    """BASELINE config-5 parameters (r=8, m=64, q=2, oversample 8, N(0,1/128)
    entries) on an n x n lattice small enough for the reference to finish."""
    return I.config5(n=n)


def cfg5_terms(n):
    """Z at the centre and ZZ on every horizontal bond (kind 0 = Z_i, 1 = Z_iZ_j;
    (kind, r0, c0, r1, c1)).  All terms live on one-row bands: the reference's
    two-row band zipper for a vertical bond needs more than 62 GB at m = 64,
    r = 8 (the golden generator was OOM-killed on it in the build container)."""
    c = n // 2 - 1
    terms = [(0, c, c, c, c)]
    terms += [(1, r, j, r, j + 1) for r in range(n) for j in range(n - 1)]
    return terms


def perturb(sites, eps, seed=1234):
    """Every site scaled elementwise by (1 + eps * xi), xi ~ N(0,1) seeded."""
    return [s * (1.0 + eps * I.gaussian(s.shape, I.derive_seed(seed, i)).real) for i, s in enumerate(sites)]


def zz_pieces(A):
    """split_two_site(Z (x) Z) pieces (observables.cpp:284-295) via the device SVD."""
    z = np.diag([1.0, -1.0]).astype(complex)
    zz = np.einsum("ac,bd->abcd", z, z)
    u, s, v = A.svd(zz.transpose(0, 2, 1, 3).copy(), 2)
    g = int((s >= 1e-14 * s[0]).sum())
    w = np.sqrt(s[:g])
    left = u.numpy()[..., :g] * w
    right = (v.numpy()[:g] * w[:, None, None]).transpose(1, 2, 0)
    return z, left, right


def device_local_expectations(A, st, opt, terms):
    """The device twin of oracle/ref_harness.cpp ref_local_expectations: cached
    environments (build_row_cache), one band environment per (r0, r1) band and a
    splice per term, each value divided by the cached norm."""
    n = st.rows
    cache = A.build_row_cache(st, opt)
    norm = A.chain_scalar(cache.tops[n - 1])
    z, left, right = zz_pieces(A)
    envs, vals = {}, []
    for kind, r0, c0, r1, c1 in terms:
        br0, br1 = min(r0, r1), max(r0, r1)
        top = cache.tops[br0 - 1] if br0 > 0 else None
        bot = cache.bots[br1 + 1] if br1 + 1 < n else None
        if (br0, br1) not in envs:
            envs[(br0, br1)] = A.band_environment(top, st, st, br0, br1, bot)
        if kind == 0:
            pieces, cc0, cc1 = [A.InsertionPiece((r0, c0), z, [])], c0, c0
        else:
            pieces = [A.InsertionPiece((r0, c0), left, [0]), A.InsertionPiece((r1, c1), right, [0])]
            cc0, cc1 = min(c0, c1), max(c0, c1)
        vals.append(A.band_splice(envs[(br0, br1)], top, st, st, bot, pieces, cc0, cc1) / norm)
    return norm, np.array(vals)
