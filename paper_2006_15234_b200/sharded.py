"""Bond-sharded two-layer row absorb: one einsumsvd per column
split across ranks along the boundary-MPS bond, collectives over
torch.distributed (NCCL between GPUs).

Reference algorithm: `two_layer_apply_row` (proj/src/contraction.cpp:254-311)
calling `einsumsvd` / `randomized_svd` (proj/src/decomposition.cpp:259-352) on
the network {v(apqsmn), S(uvst), bra*(dumbe), ket(dvncf)}, rows "apq", cols
"bctef".  The column side is sharded along t (the top-boundary bond leaving the
column); the pending tensor v, which is the previous column's t2, arrives
sharded along s.  Per rank r with t in T_r and s in S_r:

  apply  A Q:   (1) bra*(dum|be) Q_r(be|ctfX)   local
                (2) ket(vn|dcf) (1)              local
                (3) S(s|uv t_r) (2)              partial over t_r  -> all-reduce (s,n,m,X)
                (4) v_r(apq|s_r mn) (3)[s_r]     partial over s_r  -> all-reduce Y (a,p,q,X)
  adjoint A^H P: v_r^* P -> (s_r,n,m,X) -> all-gather over s; then S^*, ket^*,
                bra locally on t_r -> Z_r (b,c,t_r,e,f,X)
  big-side orth: G = all-reduce(Z_r^H Z_r) (k x k), replicated gram_factors
                (the paper's Gram-matrix orthogonalisation, Alg. 5),
                Q_r = Z_r P locally
  small side (Y, P): replicated (identical on every rank)
  projected SVD: G = all-reduce(Z_r^H Z_r), replicated eigendecomposition;
                t1 = P U w_l replicated, t2_r = conj(Z_r) conj(U) w_r / s local.

Ω_r is the t-slice of the reference's random_tensor(col_shape + [k], seed),
bit-identical to the unsharded sketch, so a sharded run reproduces the
single-device result up to the summation order of the all-reduces.  Columns
whose t extent is smaller than the world size (the last column, t = 1) run
replicated after an all-gather of v.

The compute backend is the device library (`DeviceOps`); the host code here is
only orchestration.  tests/test_sharded.py runs the same driver with a
numpy backend on world-size-2 gloo groups.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

MASK = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def _splitmix_next(state: int) -> int:
    """rng.hpp:17-23 (one step)."""
    z = (state + GAMMA) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def derive_seed(base: int, *parts: int) -> int:
    """rng.hpp:38-44: per-einsumsvd seed derive_seed(opt.seed, tag, row, col)."""
    s = base & MASK
    for p in parts:
        s = _splitmix_next((s ^ ((p + GAMMA) & MASK)) & MASK)
    return s


def shard_range(extent: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced partition of [0, extent): sizes differ by at most one."""
    base, extra = divmod(extent, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def effective_oversample(oversample: int, target: int) -> int:
    """decomposition.cpp:15-22."""
    return oversample if oversample >= 0 else max(5, int(math.ceil(0.1 * target)))


def retained_rank(s: Sequence[float], max_rank: int, rel_cutoff: float) -> int:
    """decomposition.cpp:24-29 (max_rank 0 = unbounded)."""
    if len(s) == 0:
        return 0
    floor = rel_cutoff * s[0]
    above = sum(1 for v in s if v >= floor)
    cap = len(s) if max_rank == 0 else max_rank
    return max(1, min(above, cap))


class Comm:
    """Rank / world of a torch.distributed group (world 1 when not initialised)."""

    def __init__(self, group=None):
        self.group = group
        try:
            import torch.distributed as dist
            self.dist = dist if dist.is_available() and dist.is_initialized() else None
        except Exception:  # pragma: no cover - torch without distributed
            self.dist = None
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.world = self.dist.get_world_size(group) if self.dist else 1


class DeviceOps:
    """Product backend: the device library's building blocks; collectives run
    through torch.distributed on zero-copy views of the library's buffers."""

    def __init__(self, comm: Comm, ctx=None):
        from . import api as A
        self.A = A
        self.ctx = ctx or A.default_context()
        self.comm = comm

    # --- tensors
    def shape(self, t):
        return t.shape

    def reshape(self, t, shape):
        return t.reshape(tuple(shape))

    def conj(self, t):
        return t.conj()

    def slice(self, t, axis, start, stop):
        return t.slice(axis, start, stop)

    def contract(self, spec, *ts):
        return self.A.contract(spec, *ts, ctx=self.ctx)

    def random_slice(self, shape, axis, start, stop, seed):
        return self.A.random_slice(shape, axis, start, stop - start, seed, ctx=self.ctx)

    def scale_cols(self, m, w):
        wd = self.A.to_device(np.asarray(w, dtype=np.complex128), self.ctx)
        return self.A.contract("XR,R->XR", m, wd, ctx=self.ctx)

    # --- factorizations
    def gram(self, z):
        return self.A.gram(z, self.ctx)

    def gram_factors(self, g):
        return self.A.gram_factors(g, self.ctx)

    def orth(self, y):
        return self.A.gram_orthogonalize(y, len(y.shape) - 1, self.ctx)[0]

    def projected_svd(self, z, target):
        return self.A.projected_svd(z, target, self.ctx)

    def einsumsvd(self, tensors, labels, rows, cols, max_rank, rel_cutoff, absorb, power_iters, oversample, seed):
        A = self.A
        net = A.ImplicitOperator(tensors, labels, rows, cols, ctx=self.ctx)
        r = A.einsumsvd(net, A.TruncationPolicy(max_rank, rel_cutoff), A.SvdStrategy.implicit_rsvd,
                        A.Absorb(absorb), A.RsvdConfig(power_iters, oversample, seed))
        return r.t1, r.t2, r.s

    def chain_scalar(self, sites):
        """mps.cpp:102-110 on the device."""
        t = self.A.to_device(np.ones(1, dtype=np.complex128), self.ctx)
        for s in sites:
            t = self.A.contract("l,plr->r", t, s, ctx=self.ctx)
        return complex(t.numpy()[0])

    # --- simple update (config 4)
    def exp_gate(self, op, coeff, tau):
        return self.A.hermitian_exp(op, coeff, tau, self.ctx)

    def _state(self, sites, rows, cols):
        return self.A.PepsState(rows, cols, 2, sites, ctx=self.ctx)

    def apply_one_site(self, sites, rows, cols, gate):
        out = self.A.apply_one_site(self._state(sites, rows, cols), gate,
                                    [(r, c) for r in range(rows) for c in range(cols)])
        return list(out.sites)

    def apply_two_site(self, sites, rows, cols, gate, bonds, rank):
        out = self.A.apply_two_site(self._state(sites, rows, cols), gate, bonds, self.A.TruncationPolicy(rank, 1e-14))
        return {p: out.site(*p) for bd in bonds for p in ((bd[0], bd[1]), (bd[2], bd[3]))}

    def exchange_sites(self, mine, owners):
        """Every rank's updated sites to every rank: all-gather of the shapes,
        then of the packed complex data (padded to the largest share)."""
        if self.comm.world == 1:
            return dict(mine)
        import torch
        dist, w, me = self.comm.dist, self.comm.world, self.comm.rank
        nmax = max(len(o) for o in owners)
        shp = torch.zeros(5 * max(1, nmax), dtype=torch.int64, device="cuda")
        for i, p in enumerate(owners[me]):
            shp[5 * i:5 * i + 5] = torch.tensor(mine[p].shape, dtype=torch.int64)
        shps = [torch.empty_like(shp) for _ in range(w)]
        dist.all_gather(shps, shp, group=self.comm.group)
        host = [s.cpu().numpy() for s in shps]
        sizes = [sum(int(np.prod(h[5 * i:5 * i + 5])) for i in range(len(owners[rk]))) for rk, h in enumerate(host)]
        self.ctx.sync()
        buf = torch.zeros(2 * max(1, max(sizes)), dtype=torch.float64, device="cuda")
        off = 0
        for p in owners[me]:
            x = torch.view_as_real(torch.as_tensor(mine[p], device="cuda")).reshape(-1)
            buf[off:off + x.numel()].copy_(x)
            off += x.numel()
        parts = [torch.empty_like(buf) for _ in range(w)]
        dist.all_gather(parts, buf, group=self.comm.group)
        torch.cuda.current_stream().synchronize()
        out = dict(mine)
        for rk in range(w):
            if rk == me:
                continue
            off = 0
            for i, p in enumerate(owners[rk]):
                shape = tuple(int(v) for v in host[rk][5 * i:5 * i + 5])
                n = 2 * int(np.prod(shape))
                out[p] = self.A.from_device_ptr(parts[rk][off:off + n].data_ptr(), shape, self.ctx)
                off += n
            assert off == 2 * sizes[rk]
        self.ctx.sync()
        return out

    # --- cached environments across groups
    def new_group(self, ranks):
        return self.comm.dist.new_group(ranks)

    def broadcast_boundaries(self, bounds, src):
        """Boundaries [(sites, phys)] from global rank `src` to every rank of the
        world: shapes as objects, data as NCCL broadcasts of device buffers."""
        import torch
        dist = self.comm.dist
        meta = [None if bounds is None else [([tuple(t.shape) for t in b[0]], list(b[1])) for b in bounds]]
        dist.broadcast_object_list(meta, src=src, group=self.comm.group)
        self.ctx.sync()
        out = []
        for k, (shapes, phys) in enumerate(meta[0]):
            sites = []
            for i, shp in enumerate(shapes):
                if bounds is not None:
                    x = torch.as_tensor(bounds[k][0][i], device="cuda").clone()
                else:
                    x = torch.empty(shp, dtype=torch.complex128, device="cuda")
                dist.broadcast(x, src=src, group=self.comm.group)
                torch.cuda.current_stream().synchronize()
                sites.append(self.A.from_device_ptr(x.data_ptr(), shp, self.ctx))
                self.ctx.sync()  # copied before x returns to torch's allocator
            out.append((sites, [tuple(p) for p in phys]))
        return out

    def allgather_obj(self, obj):
        out = [None] * self.comm.world
        self.comm.dist.all_gather_object(out, obj, group=self.comm.group)
        return out

    def zz_pieces(self):
        """split_two_site(Z (x) Z) (observables.cpp:284-295) with the device SVD."""
        z = np.diag([1.0, -1.0]).astype(np.complex128)
        zz = np.einsum("ac,bd->abcd", z, z)
        u, sv, v = self.A.svd(zz.transpose(0, 2, 1, 3).copy(), 2, self.ctx)
        g = retained_rank(list(sv), 4, 1e-14)
        w = np.sqrt(np.asarray(sv[:g]))
        return z, u.numpy()[..., :g] * w, (v.numpy()[:g] * w[:, None, None]).transpose(1, 2, 0)

    def band_values(self, top, bot, sites, rows, cols, r0, r1, splices):
        """One band environment (contraction.cpp:572-624) and a splice per term (:626-650)."""
        A = self.A
        st = A.PepsState(rows, cols, 2, sites, ctx=self.ctx)
        tb = A.TwoLayerBoundary.from_sites(top[0], top[1], ctx=self.ctx) if top is not None else None
        bb = A.TwoLayerBoundary.from_sites(bot[0], bot[1], ctx=self.ctx) if bot is not None else None
        env = A.band_environment(tb, st, st, r0, r1, bb)
        out = []
        for pieces, c0, c1 in splices:
            ps = [A.InsertionPiece((r, c), op, list(ids)) for r, c, op, ids in pieces]
            out.append(A.band_splice(env, tb, st, st, bb, ps, c0, c1))
        return out

    # --- collectives (in place on the library's buffer / new tensor)
    def _torch(self, t):
        import torch
        self.ctx.sync()
        return torch.as_tensor(t, device="cuda")

    def allreduce(self, t):
        if self.comm.world == 1:
            return t
        import torch
        x = self._torch(t).clone()
        self.comm.dist.all_reduce(x, group=self.comm.group)
        torch.cuda.current_stream().synchronize()
        # A fresh library tensor: its realness flag is recomputed on the summed
        # data (an in-place write would keep a stale "real" flag on `t`).
        out = self.A.from_device_ptr(x.data_ptr(), tuple(x.shape), self.ctx)
        self.ctx.sync()
        return out

    def allgather(self, t, axis, extent):
        if self.comm.world == 1:
            return t
        import torch
        x = self._torch(t)
        w = self.comm.world
        sizes = [shard_range(extent, w, r) for r in range(w)]
        mx = max(b - a for a, b in sizes)
        pad = list(x.shape)
        pad[axis] = mx
        buf = torch.zeros(pad, dtype=x.dtype, device=x.device)
        buf.narrow(axis, 0, x.shape[axis]).copy_(x)
        parts = [torch.empty_like(buf) for _ in range(w)]
        self.comm.dist.all_gather(parts, buf, group=self.comm.group)
        full = torch.cat([p.narrow(axis, 0, b - a) for p, (a, b) in zip(parts, sizes)], dim=axis).contiguous()
        torch.cuda.current_stream().synchronize()
        out = self.A.from_device_ptr(full.data_ptr(), tuple(full.shape), self.ctx)
        self.ctx.sync()  # the copy has landed before `full` returns to torch's allocator
        return out


def _absorb_weights(s, absorb):
    """decomposition.cpp:336-346 (0 split, 1 left, 2 right)."""
    s = np.asarray(s, dtype=float)
    one = np.ones_like(s)
    if absorb == 0:
        return np.sqrt(s), np.sqrt(s)
    if absorb == 1:
        return s, one
    return one, s


def sharded_column_einsumsvd(ops, v_r, S, Bc, K, s_range, T, max_rank, rel_cutoff, absorb, power_iters,
                             oversample, seed):
    """One column of the row absorb, sharded along t (see the module docstring).

    v_r: (a, p, q, s_r, m, n) local slice; S: (u, v, s, t) full; Bc = conj(bra)
    (d, u, m, b, e); K = ket (d, v, n, c, f).  Returns t1 (pb, pk, a, rank)
    replicated, t2_r (rank, b, c, t_r, e, f) local, and the kept sigma."""
    comm = ops.comm
    a, p, q, _, m_, n_ = ops.shape(v_r)
    b, e = ops.shape(Bc)[3], ops.shape(Bc)[4]
    c, f = ops.shape(K)[3], ops.shape(K)[4]
    s_full = ops.shape(S)[2]
    rows, cols = a * p * q, b * c * T * e * f
    mindim = min(rows, cols)
    target = min(max_rank if max_rank else mindim, mindim)
    probe = min(target + effective_oversample(oversample, target), mindim)
    t0, t1 = shard_range(T, comm.world, comm.rank)
    s0, s1 = s_range

    S_t = ops.slice(S, 3, t0, t1)
    S_tc = ops.conj(S_t)
    vc = ops.conj(v_r)
    Kc = ops.conj(K)
    B = ops.conj(Bc)

    def apply(x):  # x: (b, c, t_r, e, f, X) -> Y (a, p, q, X), replicated
        w1 = ops.contract("dumbe,bctefX->dumctfX", Bc, x)
        w2 = ops.contract("dvncf,dumctfX->vnumtX", K, w1)
        w3 = ops.allreduce(ops.contract("uvst,vnumtX->snmX", S_t, w2))
        w3s = ops.slice(w3, 0, s0, s1)
        return ops.allreduce(ops.contract("apqsmn,snmX->apqX", v_r, w3s))

    def adjoint(pp):  # pp: (a, p, q, X) replicated -> Z_r (b, c, t_r, e, f, X)
        r = ops.allgather(ops.contract("apqsmn,apqX->snmX", vc, pp), 0, s_full)
        w2 = ops.contract("uvst,snmX->vnumtX", S_tc, r)
        w1 = ops.contract("dvncf,vnumtX->dumctfX", Kc, w2)
        return ops.contract("dumbe,dumctfX->bctefX", B, w1)

    def orth_big(z):
        g = ops.allreduce(ops.gram(z))
        pz, _, _, _, deficient = ops.gram_factors(g)
        if np.any(deficient):  # orthonormal completion needs global rows: gather, complete, re-slice
            qf = ops.orth(ops.allgather(z, 2, T))
            return ops.slice(qf, 2, t0, t1)
        return ops.contract("bctefX,XY->bctefY", z, pz)

    omega = ops.random_slice((b, c, T, e, f, probe), 2, t0, t1, seed)
    pm = ops.orth(apply(omega))
    for _ in range(power_iters):
        qm = orth_big(adjoint(pm))
        pm = ops.orth(apply(qm))
    z = adjoint(pm)

    # projected SVD of B = P^H A = Z^H (decomposition.cpp:293-306; Gram route)
    g = ops.allreduce(ops.gram(z))
    _, _, ut, lam, _ = ops.gram_factors(g)
    s = np.sqrt(np.maximum(np.asarray(lam, dtype=float), 0.0))
    tgt = max(1, min(target, probe))
    if not (s[0] > 0.0 and s[tgt - 1] >= 1e-4 * s[0]):
        ut, s = ops.projected_svd(ops.allgather(z, 2, T), target)
    rank = min(retained_rank(list(s), max_rank, rel_cutoff), target)
    s = np.asarray(s[:rank], dtype=float)
    wl, wr = _absorb_weights(s, absorb)
    wv = np.where(s > 0.0, wr / np.where(s > 0.0, s, 1.0), 0.0)
    u_r = ops.slice(ut, 1, 0, rank)
    t1 = ops.contract("apqX,XR->pqaR", pm, ops.scale_cols(u_r, wl))
    t2 = ops.contract("bctefX,XR->Rbctef", ops.conj(z), ops.scale_cols(ops.conj(u_r), wv))
    return t1, t2, s


def sharded_two_layer_apply_row(ops, top: Sequence, top_phys: Sequence[Tuple[int, int]], bra_row: Sequence,
                                ket_row: Sequence, row: int, max_rank: int, seed: int, power_iters: int = 2,
                                oversample: int = -1, canonicalize: bool = True, seed_tag: int = 0x20,
                                rel_cutoff: float = 1e-14):
    """contraction.cpp:254-311 with every column einsumsvd sharded along the
    boundary bond.  Inputs and outputs are replicated on every rank; returns
    (sites, phys) of the new boundary."""
    comm = ops.comm
    n = len(bra_row)
    absorb = (2 if row % 2 else 1) if canonicalize else 0
    s0 = top[0]
    sh = ops.shape(s0)
    s0s = ops.reshape(s0, (top_phys[0][0], top_phys[0][1], sh[1], sh[2]))
    v = ops.contract("uvls,dumbe,dvncf->bcsef", s0s, ops.conj(bra_row[0]), ket_row[0])
    v = ops.reshape(v, (1,) + tuple(ops.shape(v)))
    sharded, s_range = False, None
    out: List = [None] * n
    for col in range(1, n):
        sc = top[col]
        sh = ops.shape(sc)
        S = ops.reshape(sc, (top_phys[col][0], top_phys[col][1], sh[1], sh[2]))
        T = sh[2]
        Bc = ops.conj(bra_row[col])
        K = ket_row[col]
        cseed = derive_seed(seed, seed_tag, row, col)
        if T >= comm.world:
            if not sharded:
                s_ext = ops.shape(v)[3]
                s_range = shard_range(s_ext, comm.world, comm.rank)
                v = ops.slice(v, 3, *s_range)
            t1, t2, _ = sharded_column_einsumsvd(ops, v, S, Bc, K, s_range, T, max_rank, rel_cutoff, absorb,
                                                 power_iters, oversample, cseed)
            v, sharded, s_range = t2, True, shard_range(T, comm.world, comm.rank)
        else:
            if sharded:
                v = ops.allgather(v, 3, ops.shape(S)[2])
                sharded = False
            t1, t2, _ = ops.einsumsvd([v, S, Bc, K], ["apqsmn", "uvst", "dumbe", "dvncf"], "apq", "bctef",
                                      max_rank, rel_cutoff, absorb, power_iters, oversample, cseed)
            t1 = ops.contract("apqR->pqaR", t1)
            v = t2
        ts = ops.shape(t1)
        out[col - 1] = ops.reshape(t1, (ts[0] * ts[1], ts[2], ts[3]))
    if sharded:
        v = ops.allgather(v, 3, ops.shape(top[n - 1])[2])
    last = ops.contract("abcdef->bcadef", v)
    ls = ops.shape(last)
    out[n - 1] = ops.reshape(last, (ls[0] * ls[1], ls[2], ls[3] * ls[4] * ls[5]))
    phys = [(ops.shape(bra_row[col])[3], ops.shape(ket_row[col])[3]) for col in range(n)]
    return out, phys


# ----------------------------------------------------------------------------- full contraction

def sharded_contract_two_layer(ops, bra_sites: Sequence, ket_sites: Sequence, rows: int, cols: int, max_rank: int,
                               seed: int, power_iters: int = 2, oversample: int = -1, canonicalize: bool = True):
    """<bra|ket> by two-layer boundary contraction (contraction.cpp:313-338:
    two_layer_first_row, then two_layer_apply_row for rows 1..n-1 with tag
    0x20, then chain_scalar mps.cpp:102-110) with every row absorb
    bond-sharded across the ranks (config 5 on N GPUs).  Sites are replicated
    (row-major list, PEPS axes (phys, up, left, down, right)); the scalar is
    returned on every rank."""
    top, phys = [], []
    for c in range(cols):
        b, k = bra_sites[c], ket_sites[c]
        sb, sk = ops.shape(b), ops.shape(k)
        t = ops.contract("dulbr,dULBR->bBlLrR", ops.conj(b), k)
        top.append(ops.reshape(t, (sb[3] * sk[3], sb[2] * sk[2], sb[4] * sk[4])))
        phys.append((sb[3], sk[3]))
    for r in range(1, rows):
        bra_row = [bra_sites[r * cols + c] for c in range(cols)]
        ket_row = [ket_sites[r * cols + c] for c in range(cols)]
        top, phys = sharded_two_layer_apply_row(ops, top, phys, bra_row, ket_row, r, max_rank, seed, power_iters,
                                                oversample, canonicalize, 0x20)
    return ops.chain_scalar(top)


# ----------------------------------------------------------------------------- cached environments

def _first_row(ops, bra_sites, ket_sites, cols):
    """two_layer_first_row (contraction.cpp:254-267), replicated."""
    top, phys = [], []
    for c in range(cols):
        b, k = bra_sites[c], ket_sites[c]
        sb, sk = ops.shape(b), ops.shape(k)
        t = ops.contract("dulbr,dULBR->bBlLrR", ops.conj(b), k)
        top.append(ops.reshape(t, (sb[3] * sk[3], sb[2] * sk[2], sb[4] * sk[4])))
        phys.append((sb[3], sk[3]))
    return top, phys


def sharded_sweep(ops, sites, rows, cols, max_rank, seed, power_iters, oversample, tag):
    """sweep_boundaries (observables.cpp:272-281) with every row absorb
    bond-sharded over ops.comm: [(sites, phys)] after rows 0..k, replicated."""
    top, phys = _first_row(ops, sites, sites, cols)
    out = [(top, phys)]
    for r in range(1, rows):
        row = [sites[r * cols + c] for c in range(cols)]
        top, phys = sharded_two_layer_apply_row(ops, top, phys, row, row, r, max_rank, seed, power_iters,
                                                oversample, True, tag)
        out.append((top, phys))
    return out


def band_groups(terms, rows):
    """Terms (kind, r0, c0, r1, c1) grouped by band (min row, max row), in band order."""
    groups = {}
    for i, (kind, r0, c0, r1, c1) in enumerate(terms):
        key = (min(r0, r1), max(r0, r1))
        if key[1] - key[0] > 1 or key[1] >= rows:
            raise ValueError("terms must lie within one row or two adjacent rows")
        groups.setdefault(key, []).append(i)
    return sorted(groups.items())


def distributed_local_expectations(ops, make_ops, sites, rows, cols, max_rank, seed, power_iters=2, oversample=-1,
                                   terms=()):
    """Cached-environment expectation values across GPU groups (
    build_row_cache observables.cpp:325-333, bands contraction.cpp:572-650).

    The world splits in two groups: the first ceil(W/2) ranks run the top sweep
    (tag 0x20), the others the bottom sweep on the vertically flipped state (tag
    0x21, bots[k] = fb[n-1-k]), each bond-sharded inside its group.  Each
    group's leader broadcasts its boundaries; the bands are then distributed by
    band row (band i on rank i mod W, one band environment + a splice per term)
    and the scalars all-gathered.  With W = 1 both sweeps run on rank 0.

    ops: the world's backend; make_ops(comm) builds one on a sub-communicator.
    terms: (kind, r0, c0, r1, c1), kind 0 = Z_i, 1 = Z_iZ_j.  Returns (norm,
    values) on every rank, values divided by the cached norm like the
    reference's expectation()."""
    comm = ops.comm
    W, me = comm.world, comm.rank
    flipped = [ops.contract("puldr->pdlur", sites[r * cols + c]) for r in range(rows - 1, -1, -1)
               for c in range(cols)]
    if W == 1:
        tops = sharded_sweep(ops, sites, rows, cols, max_rank, seed, power_iters, oversample, 0x20)
        fb = sharded_sweep(ops, flipped, rows, cols, max_rank, seed, power_iters, oversample, 0x21)
    else:
        n_top = (W + 1) // 2
        top_ranks, bot_ranks = list(range(n_top)), list(range(n_top, W))
        g_top, g_bot = ops.new_group(top_ranks), ops.new_group(bot_ranks)
        mine = g_top if me < n_top else g_bot
        sub = make_ops(Comm(mine))
        if me < n_top:
            tops = sharded_sweep(sub, sites, rows, cols, max_rank, seed, power_iters, oversample, 0x20)
            fb = None
        else:
            fb = sharded_sweep(sub, flipped, rows, cols, max_rank, seed, power_iters, oversample, 0x21)
            tops = None
        tops = ops.broadcast_boundaries(tops, 0)
        fb = ops.broadcast_boundaries(fb, n_top)
    bots = [fb[rows - 1 - k] for k in range(rows)]
    norm = ops.chain_scalar(tops[rows - 1][0])
    z, left, right = ops.zz_pieces()
    values = {}
    for bi, ((br0, br1), idx) in enumerate(band_groups(terms, rows)):
        if bi % W != me:
            continue
        top = tops[br0 - 1] if br0 > 0 else None
        bot = bots[br1 + 1] if br1 + 1 < rows else None
        splices = []
        for i in idx:
            kind, r0, c0, r1, c1 = terms[i]
            if kind == 0:
                splices.append(([(r0, c0, z, [])], c0, c0))
            else:
                splices.append(([(r0, c0, left, [0]), (r1, c1, right, [0])], min(c0, c1), max(c0, c1)))
        for i, v in zip(idx, ops.band_values(top, bot, sites, rows, cols, br0, br1, splices)):
            values[i] = v / norm
    if W > 1:
        merged = {}
        for part in ops.allgather_obj(values):
            merged.update(part)
        values = merged
    return norm, np.array([values[i] for i in range(len(terms))])


# ----------------------------------------------------------------------------- simple-update ITE

def tfim_bond_colours(rows: int, cols: int) -> List[List[Tuple[int, int, int, int]]]:
    """The four bond colours of the TFIM Trotter step in the order the driver
    applies them (csrc/ite.cpp tfim_bond_colours): even / odd horizontal, then
    even / odd vertical bonds; the bonds of one colour are disjoint."""
    out: List[List[Tuple[int, int, int, int]]] = [[], [], [], []]
    for par in range(2):
        for r in range(rows):
            for c in range(par, cols - 1, 2):
                out[par].append((r, c, r, c + 1))
    for par in range(2):
        for r in range(par, rows - 1, 2):
            for c in range(cols):
                out[2 + par].append((r, c, r + 1, c))
    return out


def sharded_ite_tfim(ops, sites: Sequence, rows: int, cols: int, J: float, h: float, tau: float, steps: int,
                     rank: int):
    """TFIM imaginary-time evolution by simple update (the reference's
    apply_ite_term loop, drivers.cpp:56-98, with apply_two_site qr_svd_gram,
    state.cpp:161-204) with the bonds of every colour split across the ranks:
    each rank updates its contiguous share of the colour's (disjoint) bonds in
    one batch, then the updated site tensors are exchanged (one all-gather of
    shapes + one of packed data per colour).  One-site field gates are applied
    replicated.  Per-bond updates are independent and deterministic, so the
    result equals the single-device / serial reference bond for bond."""
    comm = ops.comm
    x = np.array([[0, 1], [1, 0]], dtype=np.complex128)
    zz = np.diag([1.0, -1.0, -1.0, 1.0]).astype(np.complex128)
    gx = ops.exp_gate(x, -h, tau)
    gzz = ops.reshape(ops.exp_gate(zz, -J, tau), (2, 2, 2, 2))
    colours = tfim_bond_colours(rows, cols)
    sites = list(sites)
    for _ in range(steps):
        sites = ops.apply_one_site(sites, rows, cols, gx)
        for bonds in colours:
            a, b = shard_range(len(bonds), comm.world, comm.rank)
            mine = bonds[a:b]
            new = ops.apply_two_site(sites, rows, cols, gzz, mine, rank) if mine else {}
            owners = []
            for rk in range(comm.world):
                ra, rb = shard_range(len(bonds), comm.world, rk)
                owners.append([p for bd in bonds[ra:rb] for p in ((bd[0], bd[1]), (bd[2], bd[3]))])
            for (r, c), t in ops.exchange_sites(new, owners).items():
                sites[r * cols + c] = t
    return sites
