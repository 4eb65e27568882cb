"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's einsumsvd path.

This is the CPU checker, never the product: only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg may import it.  Each function restates the
reference algorithm it cites (paths relative to /root/reference/proj).  It is
pinned against the compiled reference itself (oracle/_ref, see oracle/ref.py)
by tests/test_oracle.py; BLAS/LAPACK are numpy's instead of OpenBLAS 0.3.15,
so agreement with the reference is to rounding, not bitwise, except for the
integer/RNG parts (SplitMix64, derive_seed, random_tensor) which are exact.
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

MASK = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


# ----------------------------------------------------------------------------- rng.hpp:12-44

def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix64(seed: int, n: int) -> np.ndarray:
    """First n outputs of SplitMix64(seed) (rng.hpp:17-23)."""
    with np.errstate(over="ignore"):
        i = np.arange(1, n + 1, dtype=np.uint64)
        return _mix(np.uint64(seed & MASK) + i * np.uint64(GAMMA))


def derive_seed(base: int, *parts: int) -> int:
    """rng.hpp:38-44."""
    s = base & MASK
    for p in parts:
        s = int(splitmix64((s ^ ((p + GAMMA) & MASK)) & MASK, 1)[0])
    return s


def _sym(u):
    return 2.0 * ((u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0


def random_tensor(shape, seed: int) -> np.ndarray:
    """tensor.cpp:192-201: re, im interleaved uniform on [-1, 1]."""
    n = int(np.prod(shape)) if len(shape) else 1
    u = _sym(splitmix64(seed, 2 * n))
    return (u[0::2] + 1j * u[1::2]).reshape(shape)


def random_tensor_real(shape, seed: int) -> np.ndarray:
    """tensor.cpp:203-208."""
    n = int(np.prod(shape)) if len(shape) else 1
    return _sym(splitmix64(seed, n)).astype(np.complex128).reshape(shape)


# ----------------------------------------------------------------------------- decomposition.cpp:15-29

def effective_oversample(oversample: int, target: int) -> int:
    if oversample >= 0:
        return oversample
    return max(5, int(math.ceil(0.1 * target)))


def retained_rank(s: Sequence[float], max_rank: int, rel_cutoff: float) -> int:
    if len(s) == 0:
        return 0
    floor = rel_cutoff * s[0]
    above = sum(1 for v in s if v >= floor)
    cap = len(s) if max_rank == 0 else max_rank
    return max(1, min(above, cap))


# ----------------------------------------------------------------------------- linalg.cpp

def fix_column_phases(u: np.ndarray, vt: np.ndarray | None = None):
    """linalg.cpp:44-64: largest-magnitude entry of each column real positive."""
    u = u.copy()
    vt = None if vt is None else vt.copy()
    for j in range(u.shape[1]):
        a = np.abs(u[:, j])
        i = int(np.argmax(a))  # first maximum, as the strict '>' scan
        if a[i] == 0.0:
            continue
        ph = u[i, j] / a[i]
        u[:, j] *= np.conj(ph)
        if vt is not None:
            vt[j, :] *= ph
    return u, vt


def svd(t: np.ndarray, split: int):
    """linalg.cpp:127-207 (any route computes the same thin SVD)."""
    rows = int(np.prod(t.shape[:split]))
    cols = int(np.prod(t.shape[split:]))
    u, s, vt = np.linalg.svd(t.reshape(rows, cols), full_matrices=False)
    u, vt = fix_column_phases(u, vt)
    k = s.size
    return u.reshape(t.shape[:split] + (k,)), s, vt.reshape((k,) + t.shape[split:])


def eigh(m: np.ndarray):
    """linalg.cpp:256-295: Hermiticity check, descending order, phase fix."""
    scale = np.abs(m).max() if m.size else 0.0
    if np.abs(m - m.conj().T).max() > 1e-10 * max(1.0, scale):
        raise ValueError("matrix is not Hermitian within tolerance")
    w, x = np.linalg.eigh(0.5 * (m + m.conj().T))
    w, x = w[::-1].copy(), x[:, ::-1].copy()
    x, _ = fix_column_phases(x)
    return w, x


# ----------------------------------------------------------------------------- decomposition.cpp:86-193

def _complete_deficient(q: np.ndarray, deficient: List[bool]):
    """decomposition.cpp:88-115."""
    rows, cols = q.shape
    nb = 0
    for j in range(cols):
        if not deficient[j]:
            continue
        while True:
            if nb == rows:
                raise ArithmeticError("orthonormal completion exhausted basis")
            v = np.zeros(rows, dtype=np.complex128)
            v[nb] = 1.0
            for _ in range(2):
                for c in range(cols):
                    if c == j or (deficient[c] and c > j):
                        continue
                    v = v - np.vdot(q[:, c], v) * q[:, c]
            nrm = np.linalg.norm(v)
            nb += 1
            if nrm > 0.1:
                q[:, j] = v / nrm
                break
    return q


def _gram_factors(g: np.ndarray):
    """decomposition.cpp:128-156."""
    w, x = eigh(g)
    lmax = w[0] if w.size else 0.0
    if lmax <= 0.0:
        raise ArithmeticError("gram orthogonalization of a zero operator")
    deficient = [bool(v < 1e-12 * lmax) for v in w]
    lam = np.maximum(w, 1e-12 * lmax)
    p = x / np.sqrt(lam)[None, :]
    r = np.sqrt(lam)[:, None] * x.conj().T
    return p, r, deficient


def gram_orthogonalize(a: np.ndarray, split: int):
    """decomposition.cpp:160-193."""
    rows = int(np.prod(a.shape[:split]))
    cols = int(np.prod(a.shape[split:]))
    if rows < cols:
        raise ValueError("gram orthogonalization needs row extent >= col extent")
    mat = a.reshape(rows, cols)
    p, r, deficient = _gram_factors(mat.conj().T @ mat)
    q = mat @ p
    if any(deficient):
        q = _complete_deficient(q, deficient)
    return q.reshape(a.shape[:split] + a.shape[split:]), r.reshape(a.shape[split:] + a.shape[split:])


# ----------------------------------------------------------------------------- implicit.cpp

class ImplicitOperator:
    """implicit.hpp:15-44 / implicit.cpp (contraction through np.einsum)."""

    def __init__(self, tensors, labels, rows, cols):
        self.tensors = [np.asarray(t, dtype=np.complex128) for t in tensors]
        self.labels = list(labels)
        self.rows, self.cols = rows, cols
        ext = {}
        for t, l in zip(self.tensors, self.labels):
            for c, e in zip(l, t.shape):
                ext[c] = e
        self.row_shape = tuple(ext[c] for c in rows)
        self.col_shape = tuple(ext[c] for c in cols)

    def fresh(self):
        used = self.rows + self.cols + "".join(self.labels)
        for c in "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz":
            if c not in used:
                return c
        raise ValueError("no free label")

    def apply(self, q):
        f = self.fresh()
        spec = ",".join(self.labels + [self.cols + f]) + "->" + self.rows + f
        return np.einsum(spec, *self.tensors, q, optimize="optimal")

    def adjoint_apply(self, p):
        f = self.fresh()
        spec = ",".join(self.labels + [self.rows + f]) + "->" + self.cols + f
        return np.einsum(spec, *[t.conj() for t in self.tensors], p, optimize="optimal")

    def materialize(self):
        spec = ",".join(self.labels) + "->" + self.rows + self.cols
        return np.einsum(spec, *self.tensors, optimize="optimal")


def randomized_svd(op: ImplicitOperator, max_rank: int, rel_cutoff=1e-14, power_iters=2, oversample=-1, seed=0):
    """decomposition.cpp:259-306."""
    rows, cols = int(np.prod(op.row_shape)), int(np.prod(op.col_shape))
    mindim = min(rows, cols)
    target = min(max_rank, mindim)
    clamped = max_rank > mindim
    probe = min(target + effective_oversample(oversample, target), mindim)
    q = random_tensor(op.col_shape + (probe,), seed)

    def orth(t):
        return gram_orthogonalize(t, t.ndim - 1)[0]

    p = orth(op.apply(q))
    for _ in range(power_iters):
        q = orth(op.adjoint_apply(p))
        p = orth(op.apply(q))
    b = np.moveaxis(op.adjoint_apply(p).conj(), -1, 0)
    uu, s, vv = svd(b, 1)
    u = p.reshape(rows, probe) @ uu.reshape(probe, s.size)
    rank = min(retained_rank(s, max_rank, rel_cutoff), target)
    return (u[:, :rank].reshape(op.row_shape + (rank,)), s[:rank].copy(),
            vv.reshape(s.size, cols)[:rank].reshape((rank,) + op.col_shape), clamped)


def einsumsvd(op: ImplicitOperator, max_rank: int, rel_cutoff=1e-14, strategy="implicit_rsvd", absorb="split",
              power_iters=2, oversample=-1, seed=0):
    """decomposition.cpp:308-352."""
    if strategy == "exact":
        u, s, v = svd(op.materialize(), len(op.rows))
        rank = retained_rank(s, max_rank, rel_cutoff)
        u, s, v = u[..., :rank], s[:rank], v[:rank]
        clamped = max_rank > min(int(np.prod(op.row_shape)), int(np.prod(op.col_shape)))
    else:
        u, s, v, clamped = randomized_svd(op, max_rank, rel_cutoff, power_iters, oversample, seed)
    wl = np.sqrt(s) if absorb == "split" else (s if absorb == "left" else np.ones_like(s))
    wr = np.sqrt(s) if absorb == "split" else (s if absorb == "right" else np.ones_like(s))
    return u * wl, v * wr.reshape((-1,) + (1,) * (v.ndim - 1)), s, clamped


# ----------------------------------------------------------------------------- contraction.cpp:254-338

def two_layer_first_row(sites, rows, cols):
    out, phys = [], []
    for c in range(cols):
        b = sites[c]
        t = np.einsum("dulbr,dULBR->bBlLrR", b.conj(), b)
        out.append(t.reshape(b.shape[3] ** 2, b.shape[2] ** 2, b.shape[4] ** 2))
        phys.append((b.shape[3], b.shape[3]))
    return out, phys


def two_layer_apply_row(top, phys, sites, rows, cols, row, m, seed, power_iters=2, oversample=-1,
                        canonicalize=True, tag=0x20):
    absorb = ("right" if row % 2 else "left") if canonicalize else "split"
    site = lambda r, c: sites[r * cols + c]
    s0 = top[0].reshape(phys[0][0], phys[0][1], top[0].shape[1], top[0].shape[2])
    v = np.einsum("uvls,dumbe,dvncf->bcsef", s0, site(row, 0).conj(), site(row, 0), optimize="optimal")
    v = v.reshape((1,) + v.shape)
    out = [None] * cols
    for c in range(1, cols):
        sc = top[c].reshape(phys[c][0], phys[c][1], top[c].shape[1], top[c].shape[2])
        op = ImplicitOperator([v, sc, site(row, c).conj(), site(row, c)], ["apqsmn", "uvst", "dumbe", "dvncf"],
                              "apq", "bctef")
        t1, t2, _, _ = einsumsvd(op, m if m else 2 ** 62, 1e-14, "implicit_rsvd", absorb, power_iters, oversample,
                                 derive_seed(seed, tag, row, c))
        st = t1.transpose(1, 2, 0, 3)
        out[c - 1] = st.reshape(st.shape[0] * st.shape[1], st.shape[2], st.shape[3])
        v = t2
    last = v.transpose(1, 2, 0, 3, 4, 5)
    out[cols - 1] = last.reshape(last.shape[0] * last.shape[1], last.shape[2], -1)
    newphys = [(site(row, c).shape[3], site(row, c).shape[3]) for c in range(cols)]
    return out, newphys


def chain_scalar(mps) -> complex:
    """mps.cpp:102-110."""
    t = np.ones(1, dtype=np.complex128)
    for s in mps:
        t = np.einsum("l,plr->r", t, s)
    return complex(t[0])


def contract_two_layer(sites, rows, cols, m, seed, power_iters=2, oversample=-1, canonicalize=True) -> complex:
    top, phys = two_layer_first_row(sites, rows, cols)
    for r in range(1, rows):
        top, phys = two_layer_apply_row(top, phys, sites, rows, cols, r, m, seed, power_iters, oversample,
                                        canonicalize, 0x20)
    return chain_scalar(top)


def mps_overlap(a, b) -> complex:
    """mps.cpp:112-119: <a|b>."""
    l = np.ones((1, 1), dtype=np.complex128)
    for x, y in zip(a, b):
        l = np.einsum("ab,pac,pbd->cd", l, x.conj(), y)
    return complex(l[0, 0])


def inner_exact(sites, rows, cols) -> complex:
    """Exact <psi|psi> by full dense contraction (small lattices only)."""
    return inner_exact_pair(sites, sites, rows, cols)


def inner_exact_pair(bra, ket, rows, cols) -> complex:
    """Exact <bra|ket> by full dense contraction of the merged grid
    (merge_two_layer, contraction.cpp:670-688; small lattices only)."""
    letters = iter("ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz")
    tens, specs = [], []
    hb = {}
    for r in range(rows):
        for c in range(cols):
            b, t = bra[r * cols + c], ket[r * cols + c]
            m = np.einsum("dulbr,dULBR->uUlLbBrR", b.conj(), t)
            m = m.reshape(b.shape[1] * t.shape[1], b.shape[2] * t.shape[2], b.shape[3] * t.shape[3],
                          b.shape[4] * t.shape[4])
            key_u, key_l, key_d, key_r = ("v", r, c), ("h", r, c), ("v", r + 1, c), ("h", r, c + 1)
            lab = ""
            for k in (key_u, key_l, key_d, key_r):
                if k not in hb:
                    hb[k] = next(letters)
                lab += hb[k]
            tens.append(m)
            specs.append(lab)
    return complex(np.einsum(",".join(specs) + "->", *tens, optimize="greedy"))


# ----------------------------------------------------------------------------- observables.cpp:261-333

def flip_vertical(sites, rows, cols):
    """observables.cpp:261-270: rows reversed, (phys, up, left, down, right) -> up/down swapped."""
    return [sites[r * cols + c].transpose(0, 3, 2, 1, 4) for r in range(rows - 1, -1, -1) for c in range(cols)]


def sweep_boundaries(sites, rows, cols, m, seed, power_iters=2, oversample=-1, tag=0x20):
    """observables.cpp:272-281: boundaries after rows 0..k, k = 0..rows-1."""
    top, phys = two_layer_first_row(sites, rows, cols)
    out = [(top, phys)]
    for r in range(1, rows):
        top, phys = two_layer_apply_row(top, phys, sites, rows, cols, r, m, seed, power_iters, oversample, True, tag)
        out.append((top, phys))
    return out


def build_row_cache(sites, rows, cols, m, seed, power_iters=2, oversample=-1):
    """observables.cpp:325-333: tops (tag 0x20) and bots (flipped state, tag 0x21, bots[k] = fb[n-1-k])."""
    tops = sweep_boundaries(sites, rows, cols, m, seed, power_iters, oversample, 0x20)
    fb = sweep_boundaries(flip_vertical(sites, rows, cols), rows, cols, m, seed, power_iters, oversample, 0x21)
    return tops, [fb[rows - 1 - k] for k in range(rows)]


# ----------------------------------------------------------------------------- contraction.cpp:345-650 (band zipper)

def band_value(top, bra, ket, rows, cols, r0, r1, bottom, pieces):
    """Exact contraction of band rows r0..r1 between the boundary `top` (sites,
    phys) and `bottom` (or None at the lattice edge) with insertion pieces
    [(row, col, op, bond_ids)], column by column as band_column / band_step
    build it (contraction.cpp:368-474, 545-560): carried roles [top][bra, ket per
    band row][bottom] plus the gate bonds crossing the cut."""
    if r1 < r0 or r1 - r0 > 1:
        raise ValueError("band must span one or two rows")
    IN, OUT = "ABCDEFGHIJ", "MNOPQRSTUV"
    nrows = r1 - r0 + 1
    has_top, has_bot = top is not None, bottom is not None
    roles = int(has_top) + 2 * nrows + int(has_bot)

    def partner_cols(p):
        out = {}
        for bid in p[3]:
            for q in pieces:
                if q is not p and bid in q[3]:
                    out[bid] = q[1]
        return out

    def active(c):
        ids = set()
        for p in pieces:
            for bid, pc in partner_cols(p).items():
                lo, hi = min(p[1], pc), max(p[1], pc)
                if lo <= c < hi:
                    ids.add(bid)
        return sorted(ids)

    env, env_lab, in_bonds = np.ones((), dtype=np.complex128), "", []
    for c in range(cols):
        out_bonds = active(c)
        dummies = iter("abcdefhmnopqrst")
        h_in = lambda role: next(dummies) if c == 0 else IN[role]
        h_out = lambda role: next(dummies) if c + 1 == cols else OUT[role]
        ts, labs = [env], [env_lab]
        if has_top:
            t, ph = top[0][c], top[1][c]
            ts.append(t.reshape(ph[0], ph[1], t.shape[1], t.shape[2]))
            labs.append("uv" + h_in(0) + h_out(0))
        for br in range(nrows):
            row = r0 + br
            up_b = ("u" if has_top else next(dummies)) if br == 0 else "y"
            up_k = ("v" if has_top else next(dummies)) if br == 0 else "z"
            last = br + 1 == nrows
            dn_b = ("k" if has_bot else next(dummies)) if last else "y"
            dn_k = ("l" if has_bot else next(dummies)) if last else "z"
            piece = [p for p in pieces if p[0] == row and p[1] == c]
            piece = piece[0] if piece else None
            phys_b = "w" if br == 0 else "i"
            phys_k = ("x" if br == 0 else "j") if piece else phys_b
            rb, rk = int(has_top) + 2 * br, int(has_top) + 2 * br + 1
            ts.append(bra[row * cols + c].conj())
            labs.append(phys_b + up_b + h_in(rb) + dn_b + h_out(rb))
            ts.append(ket[row * cols + c])
            labs.append(phys_k + up_k + h_in(rk) + dn_k + h_out(rk))
            if piece:
                pl = phys_b + phys_k
                pc = partner_cols(piece)
                for bid in piece[3]:
                    if pc[bid] == c:
                        pl += "g"
                    elif pc[bid] > c:
                        pl += OUT[roles + out_bonds.index(bid)]
                    else:
                        pl += IN[roles + in_bonds.index(bid)]
                ts.append(np.asarray(piece[2], dtype=np.complex128))
                labs.append(pl)
        if has_bot:
            t, ph = bottom[0][c], bottom[1][c]
            ts.append(t.reshape(ph[0], ph[1], t.shape[1], t.shape[2]))
            labs.append("kl" + h_in(roles - 1) + h_out(roles - 1))
        out_lab = (OUT[:roles] if c + 1 < cols else "") + "".join(OUT[roles + i] for i in range(len(out_bonds)))
        env = np.einsum(",".join(labs) + "->" + out_lab, *ts, optimize="optimal")
        env_lab = "".join(IN[OUT.index(ch)] for ch in out_lab)
        in_bonds = out_bonds
    return complex(env)


def zz_pieces():
    """split_two_site(Z (x) Z) (observables.cpp:284-295): SVD of op.permute{0,2,1,3}
    split 2|2, rank by retained_rank (cap d^2), sqrt(s) on both sides."""
    z = np.diag([1.0, -1.0]).astype(np.complex128)
    zz = np.einsum("ac,bd->abcd", z, z)
    u, s, vt = svd(zz.transpose(0, 2, 1, 3).copy(), 2)
    g = retained_rank(s, 4, 1e-14)
    w = np.sqrt(s[:g])
    return z, u[..., :g] * w, (vt[:g] * w[:, None, None]).transpose(1, 2, 0)


def local_expectations(sites, rows, cols, cache, terms):
    """<Z_i> / <Z_iZ_j> terms (kind, r0, c0, r1, c1) from a row cache (tops, bots),
    each band value divided by the cached norm (observables.cpp:335-422)."""
    tops, bots = cache
    norm = chain_scalar(tops[rows - 1][0])
    z, left, right = zz_pieces()
    vals = []
    for kind, r0, c0, r1, c1 in terms:
        br0, br1 = min(r0, r1), max(r0, r1)
        top = tops[br0 - 1] if br0 > 0 else None
        bot = bots[br1 + 1] if br1 + 1 < rows else None
        pieces = [(r0, c0, z, [])] if kind == 0 else [(r0, c0, left, [0]), (r1, c1, right, [0])]
        vals.append(band_value(top, sites, sites, rows, cols, br0, br1, bot, pieces) / norm)
    return norm, np.array(vals)
