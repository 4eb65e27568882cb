"""Host API mirroring the reference's public C++ interface for the einsumsvd path.

Names, argument meaning and error behaviour follow /root/reference/proj/include/peps:
``ImplicitOperator`` (implicit.hpp:15-44), ``einsumsvd`` / ``randomized_svd`` /
``gram_orthogonalize`` (decomposition.hpp:14-76), ``svd`` (linalg.hpp:15-22),
``contract`` (einsum.hpp:27), ``two_layer_first_row`` / ``two_layer_apply_row`` /
``contract_two_layer`` (contraction.hpp:77-90), ``chain_scalar`` (mps.hpp:52),
``build_row_cache`` (observables.hpp:56-61), ``band_environment`` / ``band_splice`` /
``band_value`` (contraction.hpp:95-125).  Every call goes through the C ABI of
lib/libpeps_b200.so; tensors are device-resident ``DeviceTensor`` handles (numpy
complex arrays are uploaded on the fly).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import PepsError, check, lib

_VP = C.c_void_p


class SvdStrategy(IntEnum):
    exact = 0
    implicit_rsvd = 1


class Absorb(IntEnum):
    split = 0
    left = 1
    right = 2


@dataclass
class TruncationPolicy:
    max_rank: int = 0
    rel_cutoff: float = 1e-14

    def c(self):
        return _lib.Trunc(int(self.max_rank) & 0xFFFFFFFFFFFFFFFF, float(self.rel_cutoff))


@dataclass
class RsvdConfig:
    power_iters: int = 2
    oversample: int = -1
    seed: int = 0

    def c(self):
        return _lib.Rsvd(int(self.power_iters), int(self.oversample), int(self.seed) & 0xFFFFFFFFFFFFFFFF)


@dataclass
class ContractOption:
    trunc: TruncationPolicy = field(default_factory=lambda: TruncationPolicy(0, 1e-14))
    strategy: SvdStrategy = SvdStrategy.implicit_rsvd
    rsvd: RsvdConfig = field(default_factory=RsvdConfig)
    canonicalize: bool = True
    seed: int = 0

    @staticmethod
    def two_layer_opt(m: int, seed: int = 0, power_iters: int = 2, oversample: int = -1):
        """contraction.cpp:54-62 (+ the oversample knob the configs set)."""
        return ContractOption(TruncationPolicy(m, 1e-14), SvdStrategy.implicit_rsvd,
                              RsvdConfig(power_iters, oversample, 0), True, seed)

    def c(self):
        return _lib.ContractOpt(self.trunc.c(), int(self.strategy), self.rsvd.c(), int(bool(self.canonicalize)),
                                int(self.seed) & 0xFFFFFFFFFFFFFFFF)


# ----------------------------------------------------------------------------- context

class Context:
    """One device context (stream + memory pool) of the library."""

    def __init__(self, device: int = 0):
        h = _VP()
        check(lib().pepsb_ctx_create(int(device), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().pepsb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(lib().pepsb_ctx_sync(self.h))

    def set_option(self, key: str, value: int):
        check(lib().pepsb_ctx_set_option(self.h, key.encode(), int(value)))

    def counters(self) -> dict:
        a = (C.c_uint64 * 6)()
        check(lib().pepsb_ctx_counters(self.h, a))
        return dict(flops=int(a[0]), einsumsvd_flops=int(a[1]), peak_elements=int(a[2]), launches=int(a[3]),
                    faithful_redos=int(a[4]), tsqr_fallbacks=int(a[5]))

    def counter(self, name: str) -> int:
        v = C.c_uint64()
        check(lib().pepsb_ctx_get_counter(self.h, name.encode(), C.byref(v)))
        return int(v.value)

    def reset_counters(self):
        check(lib().pepsb_ctx_reset_counters(self.h))

    def profile(self, enable: bool):
        check(lib().pepsb_ctx_profile(self.h, int(bool(enable))))

    def profile_report(self) -> dict:
        a = (C.c_double * 20)()
        check(lib().pepsb_ctx_profile_report_ex(self.h, a))
        kinds = ["gemm", "small", "gather", "other"]
        return {k: dict(launches=int(a[5 * i]), ms=a[5 * i + 1], flops=a[5 * i + 2], bytes=a[5 * i + 3],
                        exec_flops=a[5 * i + 4]) for i, k in enumerate(kinds)}

    def profile_timeline(self, cap: int = 1 << 16):
        """[(kind, start_ms, end_ms, executed_flops, side)] of the profiled launches."""
        a = (C.c_double * (5 * cap))()
        n = lib().pepsb_ctx_profile_timeline(self.h, a, cap)
        kinds = ["gemm", "small", "gather", "other"]
        return [(kinds[int(a[5 * i])], a[5 * i + 1], a[5 * i + 2], a[5 * i + 3], int(a[5 * i + 4])) for i in range(n)]

    @property
    def stream(self) -> int:
        return int(lib().pepsb_ctx_stream(self.h) or 0)


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


# ----------------------------------------------------------------------------- tensors

class DeviceTensor:
    """Device-resident complex128 tensor in the reference's row-major layout."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        try:
            if self.h:
                lib().pepsb_tensor_free(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def shape(self) -> Tuple[int, ...]:
        nd = lib().pepsb_tensor_ndim(self.h)
        s = (C.c_int64 * max(1, nd))()
        check(lib().pepsb_tensor_shape(self.h, s))
        return tuple(int(s[i]) for i in range(nd))

    @property
    def size(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1

    def numpy(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=np.complex128)
        check(lib().pepsb_tensor_to_host(self.ctx.h, self.h, out.ctypes.data_as(_VP)))
        return out

    def __repr__(self):
        return f"DeviceTensor{self.shape}"

    @property
    def data_ptr(self) -> int:
        p = _VP()
        check(lib().pepsb_tensor_data_ptr(self.h, C.byref(p)))
        return int(p.value or 0)

    @property
    def __cuda_array_interface__(self):
        """Zero-copy view for torch / NCCL (the library stream must be idle: ctx.sync())."""
        return {"shape": self.shape, "typestr": "<c16", "data": (self.data_ptr, False), "version": 3,
                "strides": None}

    def reshape(self, *shape) -> "DeviceTensor":
        if len(shape) == 1 and isinstance(shape[0], (tuple, list)):
            shape = tuple(shape[0])
        shp = (C.c_int64 * max(1, len(shape)))(*shape)
        h = _VP()
        check(lib().pepsb_tensor_reshape(self.h, len(shape), shp, C.byref(h)))
        return DeviceTensor(h, self.ctx)

    def slice(self, axis: int, start: int, stop: int) -> "DeviceTensor":
        h = _VP()
        check(lib().pepsb_tensor_slice(self.ctx.h, self.h, int(axis), int(start), int(stop - start), C.byref(h)))
        return DeviceTensor(h, self.ctx)

    def conj(self) -> "DeviceTensor":
        h = _VP()
        check(lib().pepsb_tensor_conj(self.ctx.h, self.h, C.byref(h)))
        return DeviceTensor(h, self.ctx)


def to_device(a, ctx: Optional[Context] = None) -> DeviceTensor:
    ctx = ctx or default_context()
    if isinstance(a, DeviceTensor):
        return a
    a = np.ascontiguousarray(a, dtype=np.complex128)
    shp = (C.c_int64 * max(1, a.ndim))(*a.shape)
    h = _VP()
    check(lib().pepsb_tensor_from_host(ctx.h, a.ndim, shp, a.ctypes.data_as(_VP), C.byref(h)))
    return DeviceTensor(h, ctx)


def from_device_ptr(ptr: int, shape, ctx: Optional[Context] = None) -> DeviceTensor:
    """Copy a contiguous complex128 device buffer (e.g. a torch tensor's) into a library tensor."""
    ctx = ctx or default_context()
    shp = (C.c_int64 * max(1, len(shape)))(*shape)
    h = _VP()
    check(lib().pepsb_tensor_from_device(ctx.h, len(shape), shp, _VP(int(ptr)), C.byref(h)))
    return DeviceTensor(h, ctx)


def _handles(ts, ctx):
    dts = [to_device(t, ctx) for t in ts]
    arr = (_VP * max(1, len(dts)))(*[d.h for d in dts])
    return dts, arr


def random_tensor(shape, seed: int, real: bool = False, ctx: Optional[Context] = None) -> DeviceTensor:
    """random_tensor / random_tensor_real (tensor.cpp:192-208), generated on the device."""
    ctx = ctx or default_context()
    shp = (C.c_int64 * max(1, len(shape)))(*shape)
    h = _VP()
    check(lib().pepsb_random_tensor(ctx.h, len(shape), shp, C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(real),
                                    C.byref(h)))
    return DeviceTensor(h, ctx)


def contract(spec: str, *tensors, ctx: Optional[Context] = None) -> DeviceTensor:
    ctx = ctx or default_context()
    dts, arr = _handles(tensors, ctx)
    h = _VP()
    check(lib().pepsb_contract(ctx.h, spec.encode(), len(dts), arr, C.byref(h)))
    return DeviceTensor(h, ctx)


class ImplicitOperator:
    """implicit.hpp:15-44 — a linear map given as an uncontracted network."""

    def __init__(self, tensors: Sequence, labels: Sequence[str], row_labels: str, col_labels: str,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.tensors = [to_device(t, self.ctx) for t in tensors]
        self.labels = list(labels)
        self.row_labels = row_labels
        self.col_labels = col_labels

    def _args(self):
        arr = (_VP * max(1, len(self.tensors)))(*[t.h for t in self.tensors])
        return (len(self.tensors), arr, ",".join(self.labels).encode(), self.row_labels.encode(),
                self.col_labels.encode())

    def _call(self, probe, mode):
        h = _VP()
        p = to_device(probe, self.ctx) if probe is not None else None
        check(lib().pepsb_implicit(self.ctx.h, *self._args(), p.h if p is not None else None, mode, C.byref(h)))
        return DeviceTensor(h, self.ctx)

    def apply(self, q) -> DeviceTensor:
        return self._call(q, 0)

    def adjoint_apply(self, p) -> DeviceTensor:
        return self._call(p, 1)

    def materialize(self) -> DeviceTensor:
        return self._call(None, 2)


@dataclass
class EinsumsvdResult:
    t1: DeviceTensor
    t2: DeviceTensor
    s: np.ndarray
    rank_clamped: bool


@dataclass
class SvdTriple:
    u: DeviceTensor
    s: np.ndarray
    v: DeviceTensor
    rank_clamped: bool


def einsumsvd(network: ImplicitOperator, policy: TruncationPolicy, strategy: SvdStrategy,
              absorb: Absorb = Absorb.split, cfg: RsvdConfig = RsvdConfig()) -> EinsumsvdResult:
    """decomposition.cpp:308-352."""
    ctx = network.ctx
    t1, t2 = _VP(), _VP()
    cap = 4096
    s = np.zeros(cap)
    rank = C.c_int64()
    clamped = C.c_int()
    pol, rc = policy.c(), cfg.c()
    check(lib().pepsb_einsumsvd(ctx.h, *network._args(), C.byref(pol), int(strategy), int(absorb), C.byref(rc),
                                C.byref(t1), C.byref(t2), s.ctypes.data_as(C.POINTER(C.c_double)), cap,
                                C.byref(rank), C.byref(clamped)))
    return EinsumsvdResult(DeviceTensor(t1, ctx), DeviceTensor(t2, ctx), s[:rank.value].copy(), bool(clamped.value))


def randomized_svd(op: ImplicitOperator, policy: TruncationPolicy, cfg: RsvdConfig = RsvdConfig()) -> SvdTriple:
    """decomposition.cpp:259-306."""
    ctx = op.ctx
    u, v = _VP(), _VP()
    cap = 4096
    s = np.zeros(cap)
    rank = C.c_int64()
    clamped = C.c_int()
    pol, rc = policy.c(), cfg.c()
    check(lib().pepsb_randomized_svd(ctx.h, *op._args(), C.byref(pol), C.byref(rc), C.byref(u),
                                     s.ctypes.data_as(C.POINTER(C.c_double)), cap, C.byref(rank), C.byref(v),
                                     C.byref(clamped)))
    return SvdTriple(DeviceTensor(u, ctx), s[:rank.value].copy(), DeviceTensor(v, ctx), bool(clamped.value))


def gram_orthogonalize(a, split: int, ctx: Optional[Context] = None):
    """decomposition.cpp:160-193."""
    ctx = ctx or default_context()
    d = to_device(a, ctx)
    q, r = _VP(), _VP()
    check(lib().pepsb_gram_orthogonalize(ctx.h, d.h, int(split), C.byref(q), C.byref(r)))
    return DeviceTensor(q, ctx), DeviceTensor(r, ctx)


def eigh(a, ctx: Optional[Context] = None):
    """linalg.cpp:256-295 — (values descending, vectors with phase-fixed columns)."""
    ctx = ctx or default_context()
    d = to_device(a, ctx)
    n = d.shape[0] if len(d.shape) == 2 else 0
    w = np.zeros(max(n, 1))
    v = _VP()
    check(lib().pepsb_eigh(ctx.h, d.h, w.ctypes.data_as(C.POINTER(C.c_double)), len(w), C.byref(v)))
    return w[:n].copy(), DeviceTensor(v, ctx)


def random_slice(shape, axis: int, start: int, count: int, seed: int, real: bool = False,
                 ctx: Optional[Context] = None) -> DeviceTensor:
    """Elements [start, start+count) along `axis` of random_tensor(shape, seed),
    bit-identical to slicing the full tensor (tensor.cpp:192-201 counter stream)."""
    ctx = ctx or default_context()
    shp = (C.c_int64 * max(1, len(shape)))(*shape)
    h = _VP()
    check(lib().pepsb_random_slice(ctx.h, len(shape), shp, int(axis), int(start), int(count),
                                   C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(real), C.byref(h)))
    return DeviceTensor(h, ctx)


def gram(z, ctx: Optional[Context] = None) -> DeviceTensor:
    """G = Z^H Z over the leading axes of z (last axis = probe axis)."""
    ctx = ctx or default_context()
    d = to_device(z, ctx)
    h = _VP()
    check(lib().pepsb_gram(ctx.h, d.h, C.byref(h)))
    return DeviceTensor(h, ctx)


def gram_factors(g, ctx: Optional[Context] = None):
    """decomposition.cpp:128-156 on a given Gram matrix: (P, R, X, lam, deficient)."""
    ctx = ctx or default_context()
    d = to_device(g, ctx)
    k = d.shape[0]
    lam = np.zeros(k)
    dfc = np.zeros(k, dtype=np.int32)
    p, r, x = _VP(), _VP(), _VP()
    check(lib().pepsb_gram_factors(ctx.h, d.h, C.byref(p), C.byref(r), C.byref(x),
                                   lam.ctypes.data_as(C.POINTER(C.c_double)),
                                   dfc.ctypes.data_as(C.POINTER(C.c_int)), k))
    return DeviceTensor(p, ctx), DeviceTensor(r, ctx), DeviceTensor(x, ctx), lam, dfc.astype(bool)


def projected_svd(z, target: int, ctx: Optional[Context] = None):
    """Last rSVD stage: SVD of B = Z^H -> (Ut k x k left vectors, sigma)."""
    ctx = ctx or default_context()
    d = to_device(z, ctx)
    k = d.shape[-1]
    s = np.zeros(k)
    u = _VP()
    check(lib().pepsb_projected_svd(ctx.h, d.h, int(target), C.byref(u), s.ctypes.data_as(C.POINTER(C.c_double)), k))
    return DeviceTensor(u, ctx), s


def svd(a, split: int, ctx: Optional[Context] = None):
    """linalg.cpp:193-207 — returns (u, s, v) with phase-fixed u."""
    ctx = ctx or default_context()
    d = to_device(a, ctx)
    u, v = _VP(), _VP()
    cap = 4096
    s = np.zeros(cap)
    k = C.c_int64()
    check(lib().pepsb_svd(ctx.h, d.h, int(split), C.byref(u), s.ctypes.data_as(C.POINTER(C.c_double)), cap,
                          C.byref(k), C.byref(v)))
    return DeviceTensor(u, ctx), s[:k.value].copy(), DeviceTensor(v, ctx)


# ----------------------------------------------------------------------------- PEPS level

class PepsState:
    """state.hpp:33-61 — sites (phys, up, left, down, right), row-major list."""

    def __init__(self, rows: int, cols: int, phys_dim: int, sites: Sequence, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.rows, self.cols, self.d = rows, cols, phys_dim
        self.sites = [to_device(s, self.ctx) for s in sites]
        arr = (_VP * len(self.sites))(*[s.h for s in self.sites])
        h = _VP()
        check(lib().pepsb_state_create(self.ctx.h, rows, cols, phys_dim, arr, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib().pepsb_state_free(self.h)
                self.h = None
        except Exception:
            pass

    def site(self, r, c) -> DeviceTensor:
        return self.sites[r * self.cols + c]


class TwoLayerBoundary:
    """contraction.hpp:77-80 — MPS sites (pb*pk, left, right) + phys pairs."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    @staticmethod
    def from_sites(sites: Sequence, phys: Sequence[Tuple[int, int]], ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        dts, arr = _handles(sites, ctx)
        pp = (C.c_int64 * (2 * len(phys)))(*[int(x) for p in phys for x in p])
        h = _VP()
        check(lib().pepsb_boundary_create(ctx.h, len(dts), arr, pp, C.byref(h)))
        return TwoLayerBoundary(h, ctx)

    def __del__(self):
        try:
            if self.h:
                lib().pepsb_boundary_free(self.h)
                self.h = None
        except Exception:
            pass

    def __len__(self):
        return lib().pepsb_boundary_length(self.h)

    def site(self, i) -> DeviceTensor:
        h = _VP()
        check(lib().pepsb_boundary_site(self.h, int(i), C.byref(h)))
        return DeviceTensor(h, self.ctx)

    @property
    def sites(self) -> List[DeviceTensor]:
        return [self.site(i) for i in range(len(self))]

    @property
    def phys(self) -> List[Tuple[int, int]]:
        n = len(self)
        a = (C.c_int64 * (2 * n))()
        check(lib().pepsb_boundary_phys(self.h, a))
        return [(int(a[2 * i]), int(a[2 * i + 1])) for i in range(n)]


def two_layer_first_row(bra: PepsState, ket: PepsState) -> TwoLayerBoundary:
    h = _VP()
    check(lib().pepsb_two_layer_first_row(bra.ctx.h, bra.h, ket.h, C.byref(h)))
    return TwoLayerBoundary(h, bra.ctx)


def two_layer_apply_row(top: TwoLayerBoundary, bra: PepsState, ket: PepsState, row: int, opt: ContractOption,
                        seed_tag: int = 0x20) -> TwoLayerBoundary:
    h = _VP()
    o = opt.c()
    check(lib().pepsb_two_layer_apply_row(bra.ctx.h, top.h, bra.h, ket.h, int(row), C.byref(o), C.c_uint64(seed_tag),
                                          C.byref(h)))
    return TwoLayerBoundary(h, bra.ctx)


def contract_two_layer(bra: PepsState, ket: PepsState, opt: ContractOption) -> complex:
    re, im = C.c_double(), C.c_double()
    o = opt.c()
    check(lib().pepsb_contract_two_layer(bra.ctx.h, bra.h, ket.h, C.byref(o), C.byref(re), C.byref(im)))
    return complex(re.value, im.value)


# ---- multi-GPU: NCCL communicator per context, bond-sharded row absorb

def comm_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0); broadcast the 128 bytes to the other ranks."""
    buf = C.create_string_buffer(128)
    check(lib().pepsb_comm_unique_id(buf))
    return buf.raw


def comm_init(ctx: "Context", unique_id: bytes, rank: int, world: int) -> None:
    """ncclCommInitRank on the context's device (collective over the world)."""
    if len(unique_id) != 128:
        raise ValueError("unique id must be 128 bytes")
    check(lib().pepsb_comm_init(ctx.h, unique_id, int(rank), int(world)))


def comm_init_from_torch(ctx: "Context", group=None) -> None:
    """Rank 0 draws the NCCL unique id and broadcasts it over an initialised
    torch.distributed group (any backend); every rank then joins."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    comm_init(ctx, obj[0], rank, world)


def comm_destroy(ctx: "Context") -> None:
    check(lib().pepsb_comm_destroy(ctx.h))


def two_layer_apply_row_sharded(top: TwoLayerBoundary, bra: PepsState, ket: PepsState, row: int,
                                opt: ContractOption, seed_tag: int = 0x20) -> TwoLayerBoundary:
    """two_layer_apply_row (contraction.cpp:269-311) split along the boundary
    bond across the context's communicator (C++ driver, NCCL on the library stream)."""
    h = _VP()
    o = opt.c()
    check(lib().pepsb_two_layer_apply_row_sharded(bra.ctx.h, top.h, bra.h, ket.h, int(row), C.byref(o),
                                                  C.c_uint64(seed_tag), C.byref(h)))
    return TwoLayerBoundary(h, bra.ctx)


def contract_two_layer_sharded(bra: PepsState, ket: PepsState, opt: ContractOption) -> complex:
    """contract_two_layer (contraction.cpp:313-338) with every row absorb bond-sharded."""
    re, im = C.c_double(), C.c_double()
    o = opt.c()
    check(lib().pepsb_contract_two_layer_sharded(bra.ctx.h, bra.h, ket.h, C.byref(o), C.byref(re), C.byref(im)))
    return complex(re.value, im.value)


def chain_scalar(b: TwoLayerBoundary) -> complex:
    re, im = C.c_double(), C.c_double()
    check(lib().pepsb_chain_scalar(b.ctx.h, b.h, C.byref(re), C.byref(im)))
    return complex(re.value, im.value)


def flip_vertical(s: PepsState) -> PepsState:
    """observables.cpp:261-270 — rows reversed, up/down bonds swapped."""
    h = _VP()
    check(lib().pepsb_flip_vertical(s.ctx.h, s.h, C.byref(h)))
    out = PepsState.__new__(PepsState)
    out.ctx, out.rows, out.cols, out.d, out.h = s.ctx, s.rows, s.cols, s.d, h
    out.sites = []
    for r in range(s.rows):
        for c in range(s.cols):
            t = _VP()
            check(lib().pepsb_state_site(h, r, c, C.byref(t)))
            out.sites.append(DeviceTensor(t, s.ctx))
    return out


@dataclass
class RowCache:
    tops: List[TwoLayerBoundary]
    bots: List[TwoLayerBoundary]


def build_row_cache(s: PepsState, opt: ContractOption) -> RowCache:
    h = _VP()
    o = opt.c()
    check(lib().pepsb_build_row_cache(s.ctx.h, s.h, C.byref(o), C.byref(h)))
    try:
        tops, bots = [], []
        for which, dst in ((0, tops), (1, bots)):
            for k in range(s.rows):
                b = _VP()
                check(lib().pepsb_row_cache_get(h, which, k, C.byref(b)))
                dst.append(TwoLayerBoundary(b, s.ctx))
        return RowCache(tops, bots)
    finally:
        lib().pepsb_row_cache_free(h)


@dataclass
class InsertionPiece:
    """contraction.hpp:95-99."""
    site: Tuple[int, int]
    op: object
    bond_ids: List[int] = field(default_factory=list)


class BandEnvironment:
    def __init__(self, handle, ctx):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        try:
            if self.h:
                lib().pepsb_band_env_free(self.h)
                self.h = None
        except Exception:
            pass


def _pieces(pieces: Sequence[InsertionPiece], ctx):
    n = len(pieces)
    rc = (C.c_int * max(1, 2 * n))(*[int(x) for p in pieces for x in p.site])
    ops = [to_device(p.op, ctx) for p in pieces]
    oa = (_VP * max(1, n))(*[o.h for o in ops])
    nb = (C.c_int * max(1, n))(*[len(p.bond_ids) for p in pieces])
    ids = [int(i) for p in pieces for i in p.bond_ids]
    ia = (C.c_int * max(1, len(ids)))(*ids)
    return n, rc, ops, oa, nb, ia


def band_environment(top: Optional[TwoLayerBoundary], bra: PepsState, ket: PepsState, r0: int, r1: int,
                     bottom: Optional[TwoLayerBoundary]) -> BandEnvironment:
    h = _VP()
    check(lib().pepsb_band_environment(bra.ctx.h, top.h if top else None, bra.h, ket.h, int(r0), int(r1),
                                       bottom.h if bottom else None, C.byref(h)))
    return BandEnvironment(h, bra.ctx)


def band_splice(env: BandEnvironment, top, bra: PepsState, ket: PepsState, bottom, pieces, c0: int,
                c1: int) -> complex:
    n, rc, ops, oa, nb, ia = _pieces(pieces, bra.ctx)
    re, im = C.c_double(), C.c_double()
    check(lib().pepsb_band_splice(bra.ctx.h, env.h, top.h if top else None, bra.h, ket.h,
                                  bottom.h if bottom else None, n, rc, oa, nb, ia, int(c0), int(c1), C.byref(re),
                                  C.byref(im)))
    return complex(re.value, im.value)


def band_value(top, bra: PepsState, ket: PepsState, r0: int, r1: int, bottom, pieces) -> complex:
    n, rc, ops, oa, nb, ia = _pieces(pieces, bra.ctx)
    re, im = C.c_double(), C.c_double()
    check(lib().pepsb_band_value(bra.ctx.h, top.h if top else None, bra.h, ket.h, int(r0), int(r1),
                                 bottom.h if bottom else None, n, rc, oa, nb, ia, C.byref(re), C.byref(im)))
    return complex(re.value, im.value)


def save_peps(s: PepsState, path: str) -> None:
    """save_peps (state.cpp:256-272): the reference's binary PEPS container."""
    check(lib().pepsb_save_peps(s.ctx.h, s.h, str(path).encode()))


def load_peps(path: str, ctx: Optional[Context] = None) -> PepsState:
    """load_peps (state.cpp:273-299): reads the reference's container onto the device."""
    ctx = ctx or default_context()
    h = _VP()
    check(lib().pepsb_load_peps(ctx.h, str(path).encode(), C.byref(h)))
    rows, cols, d = C.c_int(), C.c_int(), C.c_int()
    check(lib().pepsb_state_dims(h, C.byref(rows), C.byref(cols), C.byref(d)))
    out = PepsState.__new__(PepsState)
    out.ctx, out.rows, out.cols, out.d, out.h = ctx, rows.value, cols.value, d.value, h
    out.sites = []
    for r in range(out.rows):
        for c in range(out.cols):
            t = _VP()
            check(lib().pepsb_state_site(h, r, c, C.byref(t)))
            out.sites.append(DeviceTensor(t, ctx))
    return out


class ContractFamily(IntEnum):
    """contraction.hpp:14 (one-layer families)."""
    exact = 0
    bmps = 1
    ibmps = 2


def bmps_opt(m: int, seed: int = 0) -> ContractOption:
    """ContractOption::bmps_opt (contraction.cpp:36-43): exact SVD truncation."""
    return ContractOption(TruncationPolicy(m, 1e-14), SvdStrategy.exact, RsvdConfig(), True, seed)


def ibmps_opt(m: int, seed: int = 0, power_iters: int = 2, oversample: int = -1) -> ContractOption:
    """ContractOption::ibmps_opt (contraction.cpp:45-53): implicit randomized SVD."""
    return ContractOption(TruncationPolicy(m, 1e-14), SvdStrategy.implicit_rsvd, RsvdConfig(power_iters, oversample, 0),
                          True, seed)


def contract_one_layer(sites: Sequence, rows: int, cols: int, family: ContractFamily,
                       opt: Optional[ContractOption] = None, memory_budget: int = 1 << 27,
                       ctx: Optional[Context] = None) -> complex:
    """contract_one_layer (contraction.cpp:178-252) on an order-4 grid (up, left, down, right)."""
    ctx = ctx or default_context()
    dts, arr = _handles(sites, ctx)
    opt = opt or ContractOption()
    re, im = C.c_double(), C.c_double()
    o = opt.c()
    check(lib().pepsb_contract_one_layer(ctx.h, int(rows), int(cols), arr, int(family), C.byref(o),
                                         C.c_uint64(memory_budget), C.byref(re), C.byref(im)))
    return complex(re.value, im.value)


def merge_two_layer(bra: PepsState, ket: PepsState) -> List[DeviceTensor]:
    """merge_two_layer (contraction.cpp:673-688): order-4 grid of bra* x ket sites."""
    if (bra.rows, bra.cols, bra.d) != (ket.rows, ket.cols, ket.d):
        raise PepsError(2, "merge needs matching grids")
    out = []
    for b, k in zip(bra.sites, ket.sites):
        m = contract("dulbr,dULBR->uUlLbBrR", b.conj(), k, ctx=bra.ctx)
        out.append(m.reshape(b.shape[1] * k.shape[1], b.shape[2] * k.shape[2], b.shape[3] * k.shape[3],
                             b.shape[4] * k.shape[4]))
    return out


def project_to_one_layer(s: PepsState, bits: Sequence[int]) -> List[DeviceTensor]:
    """project_to_one_layer (contraction.cpp:654-671): <bits| applied on every site."""
    if len(bits) != s.rows * s.cols:
        raise PepsError(2, "bit string length must equal site count")
    out = []
    for b, t in zip(bits, s.sites):
        if not 0 <= int(b) < s.d:
            raise PepsError(2, "bit value out of range")
        e = np.zeros(s.d, dtype=np.complex128)
        e[int(b)] = 1.0
        out.append(contract("p,puldr->uldr", e, t, ctx=s.ctx))
    return out


def amplitude(s: PepsState, bits: Sequence[int], family: ContractFamily, opt: Optional[ContractOption] = None) -> complex:
    """amplitude (contraction.cpp:690-694)."""
    return contract_one_layer(project_to_one_layer(s, bits), s.rows, s.cols, family, opt, ctx=s.ctx)


def inner_product(bra: PepsState, ket: PepsState, opt: ContractOption,
                  family: Optional[ContractFamily] = None) -> complex:
    """inner_product (contraction.cpp:696-705): the two-layer IBMPS route unless a
    one-layer family (exact / bmps / ibmps) is given, which contracts the merged grid."""
    if (bra.rows, bra.cols, bra.d) != (ket.rows, ket.cols, ket.d):
        raise PepsError(2, "inner product needs matching grids")
    if family is None:
        return contract_two_layer(bra, ket, opt)
    return contract_one_layer(merge_two_layer(bra, ket), bra.rows, bra.cols, family, opt, ctx=bra.ctx)


def norm(s: PepsState, opt: ContractOption, family: Optional[ContractFamily] = None) -> float:
    """norm (contraction.cpp:707-710): sqrt(max(0, Re <s|s>))."""
    return float(np.sqrt(max(0.0, inner_product(s, s, opt, family).real)))


def approx_apply_mpo(mps: Sequence, mpo: Sequence, policy: TruncationPolicy, strategy: SvdStrategy, absorb: Absorb,
                     rsvd: RsvdConfig, seed_base: int, ctx: Optional[Context] = None) -> List[DeviceTensor]:
    """approx_apply_mpo (mps.cpp:44-84): MPS sites (phys, left, right), MPO sites (p, d, left, right)."""
    ctx = ctx or default_context()
    n = len(mps)
    ds, sa = _handles(mps, ctx)
    do, oa = _handles(mpo, ctx)
    out = (_VP * n)()
    pol, rs = policy.c(), rsvd.c()
    check(lib().pepsb_approx_apply_mpo(ctx.h, n, sa, oa, C.byref(pol), int(strategy), int(absorb), C.byref(rs),
                                       C.c_uint64(seed_base & 0xFFFFFFFFFFFFFFFF), out))
    return [DeviceTensor(out[i], ctx) for i in range(n)]


@dataclass
class LocalTerm:
    """observables.hpp:16-20: coeff * op on one or two sites; 2-site op (d,d,d,d) outputs first."""
    coeff: complex
    sites: List[Tuple[int, int]]
    op: object


@dataclass
class ExpectationOptions:
    """observables.hpp:69-77."""
    contract: ContractOption = field(default_factory=ContractOption)
    use_cache: bool = True
    shared_environments: bool = False
    allow_complex: bool = False


@dataclass
class ExpectationResult:
    """observables.hpp:79-85 (+ ExpectationStats :63-67)."""
    value: float
    raw_sum: complex
    norm_sq: float
    complex_value: complex
    full_sweeps: int
    band_contractions: int
    flops: int


def expectation(s: PepsState, terms: Sequence[LocalTerm], opt: ExpectationOptions = None) -> ExpectationResult:
    """expectation(state, observable, options) (observables.cpp:335-422) on the device."""
    from ._lib import ExpectationOpt, ExpectationResult as _R
    opt = opt or ExpectationOptions()
    n = len(terms)
    cf = (C.c_double * max(1, 2 * n))(*[x for t in terms for x in (complex(t.coeff).real, complex(t.coeff).imag)])
    ns = (C.c_int * max(1, n))(*[len(t.sites) for t in terms])
    rc = []
    for t in terms:
        flat = [int(x) for p in t.sites for x in p]
        rc += flat + [0] * (4 - len(flat))
    rca = (C.c_int * max(1, 4 * n))(*rc)
    ops = [to_device(t.op, s.ctx) for t in terms]
    oa = (_VP * max(1, n))(*[o.h for o in ops])
    o = ExpectationOpt(opt.contract.c(), int(opt.use_cache), int(opt.shared_environments), int(opt.allow_complex))
    r = _R()
    check(lib().pepsb_expectation(s.ctx.h, s.h, n, cf, ns, rca, oa, C.byref(o), C.byref(r)))
    return ExpectationResult(r.value, complex(r.raw_sum[0], r.raw_sum[1]), r.norm_sq,
                             complex(r.complex_value[0], r.complex_value[1]), int(r.full_sweeps),
                             int(r.band_contractions), int(r.flops))


def tfim_terms(rows: int, cols: int, J: float, h: float) -> List[LocalTerm]:
    """H = -J sum_<ij> Z_i Z_j - h sum_i X_i in the colour order of the ITE driver
    (fields; even / odd horizontal; even / odd vertical bonds)."""
    x = np.array([[0, 1], [1, 0]], dtype=np.complex128)
    z = np.diag([1.0, -1.0]).astype(np.complex128)
    zz = np.einsum("ac,bd->abcd", z, z)
    out = [LocalTerm(-h, [(r, c)], x) for r in range(rows) for c in range(cols)]
    for par in range(2):
        for r in range(rows):
            for c in range(par, cols - 1, 2):
                out.append(LocalTerm(-J, [(r, c), (r, c + 1)], zz))
    for par in range(2):
        for r in range(par, rows - 1, 2):
            for c in range(cols):
                out.append(LocalTerm(-J, [(r, c), (r + 1, c)], zz))
    return out


def computational_basis(rows: int, cols: int, bits: Sequence[int], d: int = 2,
                        ctx: Optional[Context] = None) -> PepsState:
    """PepsState::computational_basis (state.cpp:44-58): product state, bonds 1."""
    sites = []
    for b in bits:
        v = np.zeros((d, 1, 1, 1, 1), dtype=np.complex128)
        v[int(b), 0, 0, 0, 0] = 1.0
        sites.append(v)
    return PepsState(rows, cols, d, sites, ctx=ctx)


def run_ite(rows: int, cols: int, terms: Sequence[LocalTerm], tau: float, steps: int, evolution_rank: int,
            contraction_rank: int, rsvd_iters: int = 1, energy_every: int = 1, initial: str = "neel",
            seed: int = 0, ctx: Optional[Context] = None):
    """run_ite (drivers.cpp:75-98) on the device: per step every term in
    Hamiltonian order as exp(-tau coeff op) (apply_ite_term, drivers.cpp:56-71;
    adjacent two-site terms by the QR-reduced simple update with cap
    evolution_rank, distant ones by SWAP routing, apply_distant), runs of
    consecutive disjoint adjacent terms with the same gate
    applied in one batched call (they commute exactly); the energy
    (state_energy: cached, shared environments, two-layer IBMPS with m =
    contraction_rank, seed derive_seed(seed, 0xE, step)) every energy_every
    steps and at the end.  Returns ([(step, energy)], final state)."""
    from .inputs import derive_seed
    if tau <= 0:
        raise PepsError(5, "tau must be positive")
    if evolution_rank < 1 or contraction_rank < 1:
        raise PepsError(5, "ranks must be >= 1")
    if initial not in ("neel", "zeros"):
        raise PepsError(5, f"unknown initial state '{initial}' (use neel or zeros)")
    ctx = ctx or default_context()
    bits = [((r + c) % 2 if initial == "neel" else 0) for r in range(rows) for c in range(cols)]
    st = computational_basis(rows, cols, bits, ctx=ctx)
    d = 2
    gates = []
    for t in terms:
        op = np.asarray(t.op, dtype=np.complex128)
        if len(t.sites) == 1:
            g = hermitian_exp(op, complex(t.coeff).real, tau, ctx)
        else:
            g = hermitian_exp(op.reshape(d * d, d * d), complex(t.coeff).real, tau, ctx).reshape(d, d, d, d)
        gates.append(g)
    # batches of consecutive, site-disjoint terms sharing (op, coeff)
    groups, cur, used = [], [], set()
    key = None
    for i, t in enumerate(terms):
        k = (len(t.sites), complex(t.coeff), np.asarray(t.op).tobytes(),
             len(t.sites) == 1 or _adjacent(*t.sites))
        if complex(t.coeff).imag != 0.0:
            raise PepsError(2, "run_ite: complex term coefficients are not supported")
        sites = [tuple(p) for p in t.sites]
        if cur and (k != key or any(p in used for p in sites) or not k[3]):
            groups.append(cur)
            cur, used = [], set()
        cur.append(i)
        used.update(sites)
        key = k
    if cur:
        groups.append(cur)
    energies = []
    pol = TruncationPolicy(evolution_rank, 1e-14)
    for step in range(1, steps + 1):
        for grp in groups:
            t0 = terms[grp[0]]
            if len(t0.sites) == 1:
                st = apply_one_site(st, gates[grp[0]], [tuple(terms[i].sites[0]) for i in grp])
            elif not _adjacent(*t0.sites):  # distant: SWAP routing (one term per group)
                st = apply_distant(st, gates[grp[0]], t0.sites[0], t0.sites[1], pol)
            else:
                bonds = [tuple(terms[i].sites[0]) + tuple(terms[i].sites[1]) for i in grp]
                st = apply_two_site(st, gates[grp[0]], bonds, pol)
        if step % max(1, energy_every) == 0 or step == steps:
            opt = ExpectationOptions(ContractOption.two_layer_opt(contraction_rank, derive_seed(seed, 0xE, step),
                                                                  rsvd_iters), True, True, False)
            energies.append((step, expectation(st, terms, opt).value))
    return energies, st


SWAP = np.einsum("ad,bc->abcd", np.eye(2), np.eye(2)).astype(np.complex128)  # gates::SWAP, outputs first


def _adjacent(a, b) -> bool:
    return (a[0] == b[0] and abs(a[1] - b[1]) == 1) or (a[1] == b[1] and abs(a[0] - b[0]) == 1)


def apply_distant(s: PepsState, gate, a: Tuple[int, int], b: Tuple[int, int],
                  policy: Optional[TruncationPolicy] = None) -> PepsState:
    """apply_distant (state.cpp:206-236): route a along its row to b's column,
    then along the column, with SWAP simple updates; apply the gate on the last
    bond; route back.  Every step is the device QR-reduced simple update."""
    a, b = tuple(a), tuple(b)
    for (r, c) in (a, b):
        if not (0 <= r < s.rows and 0 <= c < s.cols):
            raise PepsError(2, f"site ({r},{c}) outside the grid")
    if a == b:
        raise PepsError(2, "distant gate needs two distinct sites")
    path = [a]
    cur = list(a)
    while cur[1] != b[1]:
        cur[1] += 1 if b[1] > cur[1] else -1
        path.append(tuple(cur))
    while cur[0] != b[0]:
        cur[0] += 1 if b[0] > cur[0] else -1
        path.append(tuple(cur))
    st = s
    for i in range(len(path) - 2):
        st = apply_two_site(st, SWAP, [path[i] + path[i + 1]], policy)
    moved = path[-2] if len(path) >= 2 else a
    st = apply_two_site(st, gate, [moved + b], policy)
    for i in range(len(path) - 3, -1, -1):
        st = apply_two_site(st, SWAP, [path[i] + path[i + 1]], policy)
    return st


def expectation_trotter(s: PepsState, terms: Sequence[LocalTerm], tau: float, opt: ExpectationOptions,
                        growth: Optional[TruncationPolicy] = None) -> float:
    """expectation_trotter (observables.cpp:424-454): <H> ~ (<psi|e^{tau H}|psi> -
    <psi|psi>) / (tau <psi|psi>), e^{tau H} applied term by term as e^{tau coeff op}
    (adjacent two-site terms by the QR-reduced simple update with the growth
    policy, which must hold the exact application: cap 0 or >= d * max_bond)."""
    if tau <= 0.0:
        raise PepsError(2, "tau must be positive")
    ctx = s.ctx
    for t in terms:  # Hermiticity as Observable::is_hermitian
        op = np.asarray(t.op, dtype=np.complex128)
        m = op.reshape(int(round(np.sqrt(op.size))), -1)
        cm = complex(t.coeff) * m
        if np.abs(cm - cm.conj().T).max() > 1e-12:
            raise PepsError(2, "Trotter expectation needs a Hermitian observable")
    growth = growth or TruncationPolicy(0, 1e-14)
    d = s.d
    phi = s
    for t in terms:
        op = np.asarray(t.op, dtype=np.complex128)
        if complex(t.coeff).imag != 0.0:
            raise PepsError(2, "expectation_trotter: complex term coefficients are not supported")
        if len(t.sites) == 1:
            phi = apply_one_site(phi, hermitian_exp(op, -complex(t.coeff).real, tau, ctx), [tuple(t.sites[0])])
        else:
            a, b = (tuple(x) for x in t.sites)
            max_bond = max(max(x.shape[1:]) for x in phi.sites)
            if growth.max_rank != 0 and growth.max_rank < d * max_bond:
                raise PepsError(2, "bond-growth policy cannot hold an exact e^{tau H_j} application")
            g = hermitian_exp(op.reshape(d * d, d * d), -complex(t.coeff).real, tau, ctx).reshape(d, d, d, d)
            phi = apply_two_site(phi, g, [a + b], growth) if _adjacent(a, b) else apply_distant(phi, g, a, b, growth)
    num = contract_two_layer(s, phi, opt.contract)
    den = contract_two_layer(s, s, opt.contract)
    return ((num - den) / (tau * den)).real


def _wrap_state(h, like: PepsState) -> PepsState:
    out = PepsState.__new__(PepsState)
    out.ctx, out.rows, out.cols, out.d, out.h = like.ctx, like.rows, like.cols, like.d, h
    out.sites = []
    for r in range(like.rows):
        for c in range(like.cols):
            t = _VP()
            check(lib().pepsb_state_site(h, r, c, C.byref(t)))
            out.sites.append(DeviceTensor(t, like.ctx))
    return out


def hermitian_exp(op, coeff: float, tau: float, ctx: Optional[Context] = None) -> DeviceTensor:
    """hermitian_function(coeff*op, exp(-tau x)) (linalg.cpp:297-314), evaluated on the device."""
    ctx = ctx or default_context()
    d = to_device(op, ctx)
    h = _VP()
    check(lib().pepsb_hermitian_exp(ctx.h, d.h, float(coeff), float(tau), C.byref(h)))
    return DeviceTensor(h, ctx)


def apply_one_site(s: PepsState, gate, sites: Sequence[Tuple[int, int]]) -> PepsState:
    """apply_one_site (state.cpp:75-85) on every listed site, one batched launch."""
    g = to_device(gate, s.ctx)
    rc = (C.c_int * max(1, 2 * len(sites)))(*[int(x) for p in sites for x in p])
    h = _VP()
    check(lib().pepsb_apply_one_site(s.ctx.h, s.h, g.h, len(sites), rc, C.byref(h)))
    return _wrap_state(h, s)


def apply_two_site(s: PepsState, gate, bonds: Sequence[Tuple[int, int, int, int]],
                   policy: Optional[TruncationPolicy] = None) -> PepsState:
    """apply_two_site (state.cpp:161-204, qr_svd_gram) on disjoint adjacent bonds (ar, ac, br, bc)."""
    g = to_device(gate, s.ctx)
    b = (C.c_int * max(1, 4 * len(bonds)))(*[int(x) for t in bonds for x in t])
    pol = (policy or TruncationPolicy(0, 1e-14)).c()
    h = _VP()
    check(lib().pepsb_apply_two_site(s.ctx.h, s.h, g.h, len(bonds), b, C.byref(pol), C.byref(h)))
    return _wrap_state(h, s)


def Ry(theta: float) -> np.ndarray:
    """gates::Ry (state.cpp:316-319): [[cos t/2, -sin t/2], [sin t/2, cos t/2]]."""
    c, s_ = np.cos(theta / 2), np.sin(theta / 2)
    return np.array([[c, -s_], [s_, c]], dtype=np.complex128)


# gates::CNOT (state.cpp:345-353): control = first site, g[c, t, c', t'] = <c t|CNOT|c' t'>
CNOT = np.zeros((2, 2, 2, 2), dtype=np.complex128)
for _c in range(2):
    for _t in range(2):
        CNOT[_c, _t ^ _c, _c, _t] = 1.0


def state_energy(s: PepsState, terms: Sequence[LocalTerm], contraction_rank: int, rsvd_iters: int,
                 seed: int) -> float:
    """state_energy (drivers.cpp:46-53) for the two-layer IBMPS family: the
    expectation with cached, shared environments (energy_contract_option,
    drivers.cpp:33-44)."""
    opt = ExpectationOptions(ContractOption.two_layer_opt(contraction_rank, seed, rsvd_iters), True, True, False)
    return expectation(s, terms, opt).value


def vqe_ansatz_state(rows: int, cols: int, layers: int, theta: Sequence[float], evolution_rank: int = 2,
                     ctx: Optional[Context] = None) -> PepsState:
    """vqe_ansatz_state (drivers.cpp:100-131): from |0...0>, per layer an Ry on
    every site (row-major), then CNOTs on every horizontal bond (row-major,
    control left) and every vertical bond (control on top), each a QR-reduced
    simple update truncated to evolution_rank (rel. cutoff 1e-14)."""
    theta = list(theta)
    if len(theta) != layers * rows * cols:
        raise PepsError(5, "theta length must be layers * rows * cols")
    st = computational_basis(rows, cols, [0] * (rows * cols), ctx=ctx)
    pol = TruncationPolicy(evolution_rank, 1e-14)
    p = 0
    for _ in range(layers):
        for r in range(rows):
            for c in range(cols):
                st = apply_one_site(st, Ry(theta[p]), [(r, c)])
                p += 1
        for r in range(rows):
            for c in range(cols - 1):
                st = apply_two_site(st, CNOT, [(r, c, r, c + 1)], pol)
        for r in range(rows - 1):
            for c in range(cols):
                st = apply_two_site(st, CNOT, [(r, c, r + 1, c)], pol)
    return st


def vqe_objective(rows: int, cols: int, layers: int, terms: Sequence[LocalTerm], evolution_rank: int = 2,
                  contraction_rank: int = 16, rsvd_iters: int = 1, seed: int = 0,
                  ctx: Optional[Context] = None):
    """The objective run_vqe minimises (drivers.cpp:166-171): theta -> energy of
    vqe_ansatz_state(theta), state_energy seeded derive_seed(seed, 0xF).  The
    host-side optimiser loop (optimize.cpp) is left to the caller."""
    from .inputs import derive_seed
    es = derive_seed(seed, 0xF)

    def f(theta):
        st = vqe_ansatz_state(rows, cols, layers, theta, evolution_rank, ctx)
        return state_energy(st, terms, contraction_rank, rsvd_iters, es)
    return f


def ite_tfim(s: PepsState, J: float, h: float, tau: float, steps: int, rank: int) -> PepsState:
    """TFIM imaginary-time evolution by batched simple update (config 4)."""
    out = _VP()
    check(lib().pepsb_ite_tfim(s.ctx.h, s.h, float(J), float(h), float(tau), int(steps), int(rank),
                               C.byref(out)))
    return _wrap_state(out, s)


__all__ = [n for n in dir() if not n.startswith("_")] + ["PepsError"]
