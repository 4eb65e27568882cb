"""Bond-sharded row absorb: the product driver
paper_2006_15234_b200/sharded.py run on world-size-2 gloo groups on CPU with a
numpy compute backend (test infrastructure: the oracle supplies the dense
kernels), against the unsharded reference restatement of two_layer_apply_row
(contraction.cpp:254-311).  Exercises even and uneven bond partitions, the
replicated edge column (t = 1) and the all-reduce / all-gather schedule."""
import os
import socket

import numpy as np
import pytest

from oracle import peps_oracle as O
from paper_2006_15234_b200 import inputs as I
from paper_2006_15234_b200 import sharded as SH


class NumpyOps:
    """Numpy backend with the DeviceOps interface (collectives over gloo)."""

    def __init__(self, comm):
        self.comm = comm
        self.calls = {"allreduce": 0, "allgather": 0}

    def shape(self, t):
        return tuple(t.shape)

    def reshape(self, t, shape):
        return np.ascontiguousarray(t).reshape(shape)

    def conj(self, t):
        return np.conj(t)

    def slice(self, t, axis, start, stop):
        return np.take(t, np.arange(start, stop), axis=axis)

    def contract(self, spec, *ts):
        return np.einsum(spec, *ts, optimize="optimal")

    def random_slice(self, shape, axis, start, stop, seed):
        return np.take(O.random_tensor(tuple(shape), seed), np.arange(start, stop), axis=axis)

    def scale_cols(self, m, w):
        return m * np.asarray(w)[None, :]

    def gram(self, z):
        zz = z.reshape(-1, z.shape[-1])
        return zz.conj().T @ zz

    def gram_factors(self, g):
        w, x = O.eigh(g)
        lmax = w[0]
        deficient = w < 1e-12 * lmax
        lam = np.maximum(w, 1e-12 * lmax)
        return x / np.sqrt(lam)[None, :], np.sqrt(lam)[:, None] * x.conj().T, x, w, deficient

    def orth(self, y):
        return O.gram_orthogonalize(y, y.ndim - 1)[0]

    def projected_svd(self, z, target):
        b = np.moveaxis(z.conj(), -1, 0)
        uu, s, _ = O.svd(b, 1)
        return uu, s

    def einsumsvd(self, tensors, labels, rows, cols, max_rank, rel_cutoff, absorb, power_iters, oversample, seed):
        op = O.ImplicitOperator(tensors, labels, rows, cols)
        t1, t2, s, _ = O.einsumsvd(op, max_rank, rel_cutoff, "implicit_rsvd", ["split", "left", "right"][absorb],
                                   power_iters, oversample, seed)
        return t1, t2, s

    def chain_scalar(self, sites):
        return O.chain_scalar(sites)

    # --- simple update: the compiled reference (oracle/_ref) as the numpy backend's kernels
    def exp_gate(self, op, coeff, tau):
        from oracle import ref
        return ref.exp_gate(op, coeff, tau)

    def apply_one_site(self, sites, rows, cols, gate):
        return [np.einsum("ij,juldr->iuldr", gate, s) for s in sites]  # state.cpp:75-85

    def apply_two_site(self, sites, rows, cols, gate, bonds, rank):
        from oracle import ref
        cur = list(sites)
        for (ar, ac, br, bc) in bonds:
            cur = ref.apply_two_site(cur, rows, cols, gate, (ar, ac), (br, bc), rank, "qr_svd_gram")
        return {p: cur[p[0] * cols + p[1]] for bd in bonds for p in ((bd[0], bd[1]), (bd[2], bd[3]))}

    def exchange_sites(self, mine, owners):
        if self.comm.world == 1:
            return dict(mine)
        import torch
        self.calls["exchange"] = self.calls.get("exchange", 0) + 1
        w, me = self.comm.world, self.comm.rank
        nmax = max(len(o) for o in owners)
        shp = torch.zeros(5 * max(1, nmax), dtype=torch.int64)
        for i, p in enumerate(owners[me]):
            shp[5 * i:5 * i + 5] = torch.tensor(mine[p].shape)
        shps = [torch.empty_like(shp) for _ in range(w)]
        self.comm.dist.all_gather(shps, shp)
        sizes = [sum(int(np.prod(h[5 * i:5 * i + 5].numpy())) for i in range(len(owners[rk])))
                 for rk, h in enumerate(shps)]
        buf = np.zeros(max(1, max(sizes)), dtype=np.complex128)
        off = 0
        for p in owners[me]:
            buf[off:off + mine[p].size] = mine[p].ravel()
            off += mine[p].size
        x = torch.from_numpy(buf.view(np.float64).copy())
        parts = [torch.empty_like(x) for _ in range(w)]
        self.comm.dist.all_gather(parts, x)
        out = dict(mine)
        for rk in range(w):
            if rk == me:
                continue
            arr = parts[rk].numpy().view(np.complex128)
            off = 0
            for i, p in enumerate(owners[rk]):
                shape = tuple(int(v) for v in shps[rk][5 * i:5 * i + 5])
                n = int(np.prod(shape))
                out[p] = arr[off:off + n].reshape(shape).copy()
                off += n
        return out

    def allreduce(self, t):
        if self.comm.world == 1:
            return t
        import torch
        self.calls["allreduce"] += 1
        x = torch.from_numpy(np.ascontiguousarray(t).view(np.float64).copy())
        self.comm.dist.all_reduce(x, group=self.comm.group)
        return x.numpy().view(np.complex128).reshape(t.shape)

    def allgather(self, t, axis, extent):
        if self.comm.world == 1:
            return t
        import torch
        self.calls["allgather"] += 1
        w = self.comm.world
        sizes = [SH.shard_range(extent, w, r) for r in range(w)]
        mx = max(b - a for a, b in sizes)
        pad = list(t.shape)
        pad[axis] = mx
        buf = np.zeros(pad, dtype=np.complex128)
        idx = [slice(None)] * t.ndim
        idx[axis] = slice(0, t.shape[axis])
        buf[tuple(idx)] = t
        x = torch.from_numpy(buf.view(np.float64).copy())
        parts = [torch.empty_like(x) for _ in range(w)]
        self.comm.dist.all_gather(parts, x, group=self.comm.group)
        out = []
        for p, (a, b) in zip(parts, sizes):
            arr = p.numpy().view(np.complex128).reshape(pad)
            idx[axis] = slice(0, b - a)
            out.append(arr[tuple(idx)])
        return np.concatenate(out, axis=axis)


    # --- cached environments across groups
    def new_group(self, ranks):
        return self.comm.dist.new_group(ranks)

    def broadcast_boundaries(self, bounds, src):
        self.calls["broadcast"] = self.calls.get("broadcast", 0) + 1
        obj = [bounds]
        self.comm.dist.broadcast_object_list(obj, src=src, group=self.comm.group)
        return obj[0]

    def allgather_obj(self, obj):
        out = [None] * self.comm.world
        self.comm.dist.all_gather_object(out, obj, group=self.comm.group)
        return out

    def zz_pieces(self):
        return O.zz_pieces()

    def band_values(self, top, bot, sites, rows, cols, r0, r1, splices):
        return [O.band_value(top, sites, sites, rows, cols, r0, r1, bot, pieces) for pieces, _, _ in splices]


def _problem(r, rows=3, cols=4, seed=11):
    sites = []
    for i in range(rows):
        for j in range(cols):
            up = 1 if i == 0 else r
            left = 1 if j == 0 else r
            down = 1 if i == rows - 1 else r
            right = 1 if j == cols - 1 else r
            sites.append(O.random_tensor((2, up, left, down, right), O.derive_seed(seed, i, j)))
    top, phys = O.two_layer_first_row(sites, rows, cols)
    return sites, top, phys


def _run_sharded(ops, r, m, row=1, rows=3, cols=4, oversample=-1):
    sites, top, phys = _problem(r, rows, cols)
    bra = [sites[row * cols + c] for c in range(cols)]
    got, gphys = SH.sharded_two_layer_apply_row(ops, top, phys, bra, bra, row, m, 7, 2, oversample, True, 0x20)
    ref, rphys = O.two_layer_apply_row(top, phys, sites, rows, cols, row, m, 7, 2, oversample, True, 0x20)
    assert [tuple(p) for p in gphys] == [tuple(p) for p in rphys]
    err = 0.0
    for a, b in zip(got, ref):
        assert a.shape == b.shape
        err = max(err, float(np.abs(a - b).max() / np.abs(b).max()))
    return err


def test_shard_ranges_partition():
    for extent in (1, 4, 9, 64):
        for world in (1, 2, 3, 8):
            rs = [SH.shard_range(extent, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == extent
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_derive_seed_matches_reference_rng():
    for parts in [(0x20, 1, 2), (0x21, 5, 9), (1,), ()]:
        assert SH.derive_seed(123456789, *parts) == O.derive_seed(123456789, *parts)


@pytest.mark.parametrize("r,m", [(2, 4), (3, 6)])
def test_sharded_row_world1(r, m):
    err = _run_sharded(NumpyOps(SH.Comm()), r, m)
    assert err < 1e-9


def _worker(rank, world, port, r, m, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = NumpyOps(SH.Comm())
        err = _run_sharded(ops, r, m)
        q.put((rank, err, dict(ops.calls)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("r,m", [(2, 4), (3, 6)])
def test_sharded_row_world2_gloo(r, m):
    """r = 2: bond t = 4 split 2 + 2; r = 3: t = 9 split 5 + 4 (uneven)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, 2, port, r, m, q)) for rk in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = [q.get(timeout=5) for _ in procs]
    for rank, err, calls in res:
        assert err < 1e-9, (rank, err)
        # two sharded columns (q = 2): per column 2 all-reduces per apply x 3 applies,
        # 1 all-gather per adjoint x 3, Gram all-reduces, plus the v gather before the edge column
        assert calls["allreduce"] >= 2 * (2 * 3 + 3) and calls["allgather"] >= 2 * 3 + 1


# ----------------------------------------------------------------------------- full contraction / ITE

def _contract_case(ops, r=2, m=4, rows=4, cols=3):
    sites, _, _ = _problem(r, rows, cols, seed=23)
    got = SH.sharded_contract_two_layer(ops, sites, sites, rows, cols, m, 5, 2, -1, True)
    want = O.contract_two_layer(sites, rows, cols, m, 5, 2, -1, True)
    return abs(got - want) / abs(want)


def _ite_case(ops, rows=3, cols=4, steps=3, rank=3):
    from oracle import ref
    plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(rows * cols)]
    got = SH.sharded_ite_tfim(ops, plus, rows, cols, 1.0, 3.0, 0.05, steps, rank)
    want, _ = ref.ite_tfim(plus, rows, cols, 1.0, 3.0, 0.05, steps, rank)
    assert [g.shape for g in got] == [w.shape for w in want]
    return max(float(np.abs(g - w).max() / np.abs(w).max()) for g, w in zip(got, want))


def test_tfim_bond_colours_disjoint_and_complete():
    cols = SH.tfim_bond_colours(3, 4)
    allb = [b for c in cols for b in c]
    assert len(allb) == len(set(allb)) == 3 * 3 + 2 * 4
    for c in cols:
        sites = [p for b in c for p in ((b[0], b[1]), (b[2], b[3]))]
        assert len(sites) == len(set(sites))


def test_sharded_contract_world1():
    assert _contract_case(NumpyOps(SH.Comm())) < 1e-9


def _worker2(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = NumpyOps(SH.Comm())
        e1 = _contract_case(ops)
        e2 = _ite_case(ops)
        q.put((rank, e1, e2, dict(ops.calls)))
    finally:
        dist.destroy_process_group()


def test_sharded_contract_and_ite_world2_gloo(refo):
    """Config-5 style norm (every row absorb bond-sharded) and config-4 style
    simple-update ITE with each colour's bonds split across 2 ranks and the
    updated sites exchanged, against the serial reference."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker2, args=(rk, 2, port, q)) for rk in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = [q.get(timeout=5) for _ in procs]
    for rank, e1, e2, calls in res:
        assert e1 < 1e-9, (rank, e1)
        assert e2 < 1e-12, (rank, e2)  # per-bond updates are the reference's own code
        assert calls["exchange"] == 3 * 4  # one exchange per colour per step


# ----------------------------------------------------------------------------- cached environments across groups

def _cache_terms(rows, cols):
    terms = [(0, i // cols, i % cols, i // cols, i % cols) for i in range(rows * cols)]
    terms += [(1, 1, 1, 1, 2), (1, 0, 2, 1, 2), (1, 2, 3, 3, 3), (1, 3, 0, 3, 1)]
    return terms


def _cache_case(ops, make_ops):
    """Config-3/5 style: <Z_i> on every site + horizontal / vertical ZZ from the
    distributed cached environments, against the reference's own values
    (tests/golden/golden.npz: bands_*, generated by oracle/_ref) and the serial
    numpy restatement."""
    import numpy as _np
    sites = I.random_peps(4, 4, 2, 91, scale=1 / _np.sqrt(8))
    terms = _cache_terms(4, 4)
    norm, vals = SH.distributed_local_expectations(ops, make_ops, sites, 4, 4, 4, 13, 2, -1, terms)
    g = dict(_np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")))
    assert [tuple(t) for t in g["bands_terms"]] == terms
    return abs(norm - g["bands_norm"][0]) / abs(g["bands_norm"][0]), float(_np.abs(vals - g["bands_values"]).max())


def test_numpy_band_restatement_matches_reference_golden(golden):
    sites = I.random_peps(4, 4, 2, 91, scale=1 / np.sqrt(8))
    cache = O.build_row_cache(sites, 4, 4, 4, 13, 2, -1)
    norm, vals = O.local_expectations(sites, 4, 4, cache, [tuple(t) for t in golden["bands_terms"]])
    assert abs(norm - golden["bands_norm"][0]) <= 1e-12 * abs(golden["bands_norm"][0])
    assert np.abs(vals - golden["bands_values"]).max() < 1e-12


def test_distributed_cache_world1():
    en, ev = _cache_case(NumpyOps(SH.Comm()), NumpyOps)
    assert en < 1e-10 and ev < 1e-10


def _worker3(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = NumpyOps(SH.Comm())
        made = []

        def make_ops(comm):
            made.append(NumpyOps(comm))
            return made[-1]

        en, ev = _cache_case(ops, make_ops)
        sub = made[0].calls if made else {}
        q.put((rank, en, ev, dict(ops.calls), dict(sub), made[0].comm.world if made else 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_cache_gloo(world):
    """SURVEY §8(e) row 2 on world-size-2 and -3 gloo groups: the top and bottom
    sweeps on separate rank groups (bond-sharded inside a group of 2 at world
    3), boundaries broadcast, bands distributed by row, scalars gathered; norm
    and all 20 values match the reference to 1e-10 on every rank."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker3, args=(rk, world, port, q)) for rk in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = [q.get(timeout=5) for _ in procs]
    for rank, en, ev, calls, sub, sub_world in res:
        assert en < 1e-10 and ev < 1e-10, (rank, en, ev)
        assert calls["broadcast"] == 2  # tops from rank 0, bots from the bottom group's leader
        assert sub_world == (((world + 1) // 2) if rank < (world + 1) // 2 else world // 2)
        if sub_world > 1:  # the sweep inside a group is itself bond-sharded
            assert sub["allreduce"] > 0 and sub["allgather"] > 0
