"""TEST INFRASTRUCTURE ONLY — ctypes view of the reference oracle.

Loads ``oracle/_ref/libpeps_ref.so`` (the unmodified reference sources under
/root/reference/proj/src compiled by ``oracle/Makefile`` plus
``oracle/ref_harness.cpp``) and exposes the reference's public API on numpy
complex128 arrays.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline legs may import this module; the product path
(``paper_2006_15234_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libpeps_ref.so")

_lib = None


class RefError(RuntimeError):
    """Mirrors the reference exception family (errors.hpp:10-34)."""

    KINDS = {1: "ShapeError", 2: "ValidationError", 3: "ResourceError", 4: "NumericalError",
             5: "ConfigError", 9: "Error"}

    def __init__(self, kind: int, msg: str):
        super().__init__(f"{self.KINDS.get(kind, 'Error')}: {msg}")
        self.kind = self.KINDS.get(kind, "Error")


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_derive_seed.restype = C.c_uint64
        _lib.ref_flops.restype = C.c_uint64
        _lib.ref_einsumsvd_flops.restype = C.c_uint64
        _lib.ref_peak_elements.restype = C.c_uint64
        for name in dir(_lib):
            pass
    return _lib


def _fn(name):
    f = getattr(lib(), name)
    f.restype = C.c_void_p
    return f


# ----------------------------------------------------------------------------- marshalling

class _TList:
    """Keeps a list of complex arrays alive and exposes (nt, ndims, shapes, datas)."""

    def __init__(self, arrays: Sequence[np.ndarray]):
        self.arrays = [np.ascontiguousarray(a, dtype=np.complex128) for a in arrays]
        self.nt = len(self.arrays)
        self.ndims = (C.c_int * max(1, self.nt))(*[a.ndim for a in self.arrays])
        shp = [int(e) for a in self.arrays for e in a.shape]
        self.shapes = (C.c_int64 * max(1, len(shp)))(*shp)
        self.datas = (C.c_void_p * max(1, self.nt))(*[a.ctypes.data for a in self.arrays])

    def args(self):
        return (self.nt, self.ndims, self.shapes, self.datas)


def _bag(ptr):
    L = lib()
    if not ptr:
        raise RefError(L.ref_last_error_type(), L.ref_last_error().decode())
    bag = C.c_void_p(ptr)
    try:
        nt = L.ref_bag_ntensors(bag)
        tensors = []
        for i in range(nt):
            nd = L.ref_bag_tensor_ndim(bag, i)
            shp = (C.c_int64 * max(1, nd))()
            L.ref_bag_tensor_shape(bag, i, shp)
            shape = tuple(int(shp[j]) for j in range(nd))
            out = np.empty(shape, dtype=np.complex128)
            L.ref_bag_tensor_data(bag, i, C.c_void_p(out.ctypes.data))
            tensors.append(out)
        nd = L.ref_bag_ndoubles(bag)
        dbl = np.empty(nd, dtype=np.float64)
        if nd:
            L.ref_bag_doubles(bag, C.c_void_p(dbl.ctypes.data))
        return tensors, dbl
    finally:
        L.ref_bag_free(bag)


def _i64(vals):
    vals = [int(v) for v in vals]
    return (C.c_int64 * max(1, len(vals)))(*vals)


# ----------------------------------------------------------------------------- API

def set_threads(n: int) -> None:
    lib().ref_set_threads(int(n))


def reset_counters() -> None:
    lib().ref_reset_counters()


def flops() -> int:
    return int(lib().ref_flops())


def derive_seed(base: int, *parts: int) -> int:
    arr = (C.c_uint64 * max(1, len(parts)))(*[p & 0xFFFFFFFFFFFFFFFF for p in parts])
    return int(lib().ref_derive_seed(C.c_uint64(base & 0xFFFFFFFFFFFFFFFF), len(parts), arr))


def random_tensor(shape, seed: int, real: bool = False) -> np.ndarray:
    t, _ = _bag(_fn("ref_random_tensor")(len(shape), _i64(shape), C.c_uint64(seed), int(real)))
    return t[0]


def contract(spec: str, *tensors) -> np.ndarray:
    tl = _TList(tensors)
    t, _ = _bag(_fn("ref_contract")(spec.encode(), *tl.args()))
    return t[0]


def _net(tensors, labels, rows, cols):
    tl = _TList(tensors)
    return tl, ",".join(labels).encode(), rows.encode(), cols.encode()


def implicit_apply(tensors, labels, rows, cols, probe, adjoint=False, timed=False):
    """ImplicitOperator::apply / adjoint_apply (implicit.cpp:66-100); with
    timed=True also the seconds the reference spent inside the call (operator
    construction and host marshalling excluded)."""
    tl, lab, r, c = _net(tensors, labels, rows, cols)
    p = np.ascontiguousarray(probe, dtype=np.complex128)
    t, d = _bag(_fn("ref_implicit")(1 if adjoint else 0, *tl.args(), lab, r, c, p.ndim,
                                    _i64(p.shape), C.c_void_p(p.ctypes.data)))
    return (t[0], float(d[0])) if timed else t[0]


def materialize(tensors, labels, rows, cols):
    tl, lab, r, c = _net(tensors, labels, rows, cols)
    t, _ = _bag(_fn("ref_implicit")(2, *tl.args(), lab, r, c, 0, None, None))
    return t[0]


STRATEGY = {"exact": 0, "implicit_rsvd": 1}
ABSORB = {"split": 0, "left": 1, "right": 2}


def einsumsvd(tensors, labels, rows, cols, max_rank, rel_cutoff=1e-14, strategy="implicit_rsvd",
              absorb="split", power_iters=2, oversample=-1, seed=0):
    """Returns dict(t1, t2, s, rank_clamped, seconds, flops) — decomposition.cpp:308-352."""
    tl, lab, r, c = _net(tensors, labels, rows, cols)
    t, d = _bag(_fn("ref_einsumsvd")(*tl.args(), lab, r, c, C.c_uint64(max_rank),
                                     C.c_double(rel_cutoff), STRATEGY[strategy], ABSORB[absorb],
                                     int(power_iters), int(oversample), C.c_uint64(seed)))
    return dict(t1=t[0], t2=t[1], s=d[:-3].copy(), rank_clamped=bool(d[-3]), seconds=float(d[-2]),
                flops=float(d[-1]))


def randomized_svd(tensors, labels, rows, cols, max_rank, rel_cutoff=1e-14, power_iters=2,
                   oversample=-1, seed=0):
    tl, lab, r, c = _net(tensors, labels, rows, cols)
    t, d = _bag(_fn("ref_randomized_svd")(*tl.args(), lab, r, c, C.c_uint64(max_rank),
                                          C.c_double(rel_cutoff), int(power_iters),
                                          int(oversample), C.c_uint64(seed)))
    return dict(u=t[0], v=t[1], s=d[:-1].copy(), rank_clamped=bool(d[-1]))


def gram_orthogonalize(a, split):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    t, _ = _bag(_fn("ref_gram_orthogonalize")(a.ndim, _i64(a.shape), C.c_void_p(a.ctypes.data),
                                              int(split)))
    return t[0], t[1]


def svd(a, split):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    t, d = _bag(_fn("ref_svd")(a.ndim, _i64(a.shape), C.c_void_p(a.ctypes.data), int(split)))
    return t[0], d, t[1]


def eigh(m):
    m = np.ascontiguousarray(m, dtype=np.complex128)
    t, d = _bag(_fn("ref_eigh")(m.shape[0], C.c_void_p(m.ctypes.data)))
    return d, t[0]


# ----------------------------------------------------------------------------- PEPS level

def _state_args(sites, rows, cols, d):
    tl = _TList(sites)
    return tl, (rows, cols, d, tl.ndims, tl.shapes, tl.datas)


def two_layer_first_row(sites, rows, cols, d=2):
    tl, a = _state_args(sites, rows, cols, d)
    t, dd = _bag(_fn("ref_two_layer_first_row")(*a))
    return t, [(int(dd[2 * i]), int(dd[2 * i + 1])) for i in range(cols)]


def two_layer_apply_row(top_sites, phys, sites, rows, cols, row, m, seed, power_iters=2,
                        oversample=-1, canonicalize=True, tag=0x20, d=2):
    tl, a = _state_args(sites, rows, cols, d)
    top = _TList(top_sites)
    pp = _i64([x for p in phys for x in p])
    t, dd = _bag(_fn("ref_two_layer_apply_row")(*a, top.ndims, top.shapes, top.datas, pp, int(row),
                                                C.c_int64(m), C.c_uint64(seed), int(power_iters),
                                                int(oversample), int(canonicalize),
                                                C.c_uint64(tag)))
    phys_out = [(int(dd[2 * i]), int(dd[2 * i + 1])) for i in range(cols)]
    return t, phys_out, dict(seconds=float(dd[-2]), flops=float(dd[-1]))


def contract_two_layer(sites, rows, cols, m, seed, power_iters=2, oversample=-1, canonicalize=True,
                       d=2):
    tl, a = _state_args(sites, rows, cols, d)
    _, dd = _bag(_fn("ref_contract_two_layer")(*a, C.c_int64(m), C.c_uint64(seed),
                                               int(power_iters), int(oversample),
                                               int(canonicalize)))
    return complex(dd[0], dd[1]), dict(seconds=float(dd[2]), flops=float(dd[3]), peak=float(dd[4]))


def save_peps(sites, rows, cols, path, d=2):
    tl, a = _state_args(sites, rows, cols, d)
    _bag(_fn("ref_save_peps")(*a, str(path).encode()))


def load_peps(path):
    t, dd = _bag(_fn("ref_load_peps")(str(path).encode()))
    return t, int(dd[0]), int(dd[1]), int(dd[2])


def contract_one_layer(sites, rows, cols, family, m=0, seed=0, power_iters=2, oversample=-1, canonicalize=True):
    """contract_one_layer on an order-4 grid; family 0 exact, 1 bmps, 2 ibmps."""
    tl = _TList(sites)
    _, dd = _bag(_fn("ref_contract_one_layer")(int(rows), int(cols), tl.ndims, tl.shapes, tl.datas, int(family),
                                               C.c_int64(m),
                                               C.c_uint64(seed), int(power_iters), int(oversample),
                                               int(canonicalize)))
    return complex(dd[0], dd[1])


def inner_exact(sites, rows, cols, d=2):
    tl, a = _state_args(sites, rows, cols, d)
    _, dd = _bag(_fn("ref_inner_exact")(*a))
    return complex(dd[0], dd[1])


def local_expectations(sites, rows, cols, m, seed, terms, power_iters=2, oversample=-1, d=2):
    """terms: list of (kind, r0, c0, r1, c1); kind 0 = Z_i, 1 = Z_iZ_j."""
    tl, a = _state_args(sites, rows, cols, d)
    flat = (C.c_int * max(1, 5 * len(terms)))(*[int(x) for t in terms for x in t])
    _, dd = _bag(_fn("ref_local_expectations")(*a, C.c_int64(m), C.c_uint64(seed),
                                               int(power_iters), int(oversample), len(terms), flat))
    norm = complex(dd[0], dd[1])
    vals = dd[2:2 + 2 * len(terms)].reshape(-1, 2)
    return norm, vals[:, 0] + 1j * vals[:, 1], dict(t_cache=float(dd[-2]), t_bands=float(dd[-1]))


def tfim_energy(sites, rows, cols, J, h, m, seed, power_iters=2, oversample=-1, shared_env=True,
                d=2):
    tl, a = _state_args(sites, rows, cols, d)
    _, dd = _bag(_fn("ref_tfim_energy")(*a, C.c_double(J), C.c_double(h), C.c_int64(m),
                                        C.c_uint64(seed), int(power_iters), int(oversample),
                                        int(shared_env)))
    return dict(value=float(dd[0]), norm_sq=float(dd[1]), raw_sum=complex(dd[2], dd[3]))


UPDATE = {"direct": 0, "qr_svd": 1, "qr_svd_gram": 2}


def apply_two_site(sites, rows, cols, gate, a, b, max_rank=0, strategy="qr_svd_gram", d=2):
    tl, args = _state_args(sites, rows, cols, d)
    g = np.ascontiguousarray(gate, dtype=np.complex128)
    t, _ = _bag(_fn("ref_apply_two_site")(*args, C.c_void_p(g.ctypes.data), int(a[0]), int(a[1]),
                                          int(b[0]), int(b[1]), C.c_uint64(max_rank),
                                          UPDATE[strategy]))
    return t


def exp_gate(op, coeff, tau):
    op = np.ascontiguousarray(op, dtype=np.complex128)
    t, _ = _bag(_fn("ref_exp_gate")(op.shape[0], C.c_void_p(op.ctypes.data), C.c_double(coeff),
                                    C.c_double(tau)))
    return t[0]


def ite_tfim(sites, rows, cols, J, h, tau, steps, rank, d=2):
    tl, a = _state_args(sites, rows, cols, d)
    t, dd = _bag(_fn("ref_ite_tfim")(*a, C.c_double(J), C.c_double(h), C.c_double(tau),
                                     int(steps), C.c_uint64(rank)))
    return t, float(dd[0])


def run_ite(rows, cols, J, h, tau, steps, evolution_rank, contraction_rank, rsvd_iters=1, energy_every=1,
            initial="neel", seed=0):
    """run_ite (drivers.cpp:75-98), TFIM in colour order: ([(step, energy)], final sites)."""
    t, dd = _bag(_fn("ref_run_ite")(int(rows), int(cols), C.c_double(J), C.c_double(h), C.c_double(tau),
                                    int(steps), C.c_uint64(evolution_rank), C.c_uint64(contraction_rank),
                                    int(rsvd_iters), int(energy_every), int(initial == "neel"),
                                    C.c_uint64(seed)))
    e = [(int(dd[2 * i]), float(dd[2 * i + 1])) for i in range(len(dd) // 2)]
    return e, t


def vqe_ansatz(rows, cols, layers, theta, evolution_rank, J, h, contraction_rank, rsvd_iters, seed):
    """vqe_ansatz_state (drivers.cpp:100-131) + its TFIM energy (run_vqe objective): (sites, energy)."""
    th = np.ascontiguousarray(theta, dtype=np.float64)
    t, dd = _bag(_fn("ref_vqe_ansatz")(int(rows), int(cols), int(layers), C.c_void_p(th.ctypes.data),
                                       C.c_uint64(evolution_rank), C.c_double(J), C.c_double(h),
                                       C.c_uint64(contraction_rank), int(rsvd_iters), C.c_uint64(seed)))
    return t, float(dd[0])


def apply_distant(sites, rows, cols, gate, a, b, max_rank=0, d=2):
    tl, args = _state_args(sites, rows, cols, d)
    g = np.ascontiguousarray(gate, dtype=np.complex128)
    t, _ = _bag(_fn("ref_apply_distant")(*args, C.c_void_p(g.ctypes.data), int(a[0]), int(a[1]), int(b[0]),
                                         int(b[1]), C.c_uint64(max_rank)))
    return t


def expectation_trotter(sites, rows, cols, J, h, tau, m, seed, power_iters=2, oversample=-1, growth_cap=0, d=2):
    tl, a = _state_args(sites, rows, cols, d)
    _, dd = _bag(_fn("ref_expectation_trotter")(*a, C.c_double(J), C.c_double(h), C.c_double(tau), C.c_int64(m),
                                                C.c_uint64(seed), int(power_iters), int(oversample),
                                                C.c_uint64(growth_cap)))
    return float(dd[0])


def plus_state(rows, cols):
    t, _ = _bag(_fn("ref_plus_state")(int(rows), int(cols)))
    return t


def chain_scalar(sites):
    tl = _TList(sites)
    _, dd = _bag(_fn("ref_chain_scalar")(*tl.args()))
    return complex(dd[0], dd[1])


def json_driver(which: str, config: str) -> str:
    """run_expect_json / run_vqe_json / run_ite_json (drivers.cpp:265-550): the result document."""
    L = lib()
    L.ref_bag_text_len.restype = C.c_int64
    ptr = _fn("ref_json_driver")({"expect": 0, "vqe": 1, "ite": 2}[which], config.encode())
    if not ptr:
        raise RefError(L.ref_last_error_type(), L.ref_last_error().decode())
    bag = C.c_void_p(ptr)
    try:
        n = L.ref_bag_text_len(bag)
        buf = C.create_string_buffer(int(n) + 1)
        L.ref_bag_text(bag, buf)
        return buf.raw[:n].decode()
    finally:
        L.ref_bag_free(bag)


def minimize(method: str, fn: int, x0, max_evaluations=300, tolerance=1e-6, initial_step=0.4):
    """optimize.cpp minimize on analytic objective `fn` (0 Rosenbrock, 1 quadratic + cosine)."""
    x = np.ascontiguousarray(x0, dtype=np.float64)
    t, d = _bag(_fn("ref_minimize")(method.encode(), int(fn), len(x), C.c_void_p(x.ctypes.data),
                                    int(max_evaluations), C.c_double(tolerance), C.c_double(initial_step)))
    return dict(converged=bool(d[0]), evaluations=int(d[1]), best_f=float(d[2]), trace=d[3:].copy(),
                best_x=t[0].real.copy())


def band_environment_time(top_sites, top_phys, bot_sites, bot_phys, sites, rows, cols, r0, r1, d=2):
    """Seconds of one band_environment (contraction.cpp:572-624) on the reference."""
    tl, a = _state_args(sites, rows, cols, d)
    top, bot = _TList(top_sites), _TList(bot_sites)
    _, dd = _bag(_fn("ref_band_environment_time")(*a, top.ndims, top.shapes, top.datas,
                                                  _i64([x for p in top_phys for x in p]), bot.ndims, bot.shapes,
                                                  bot.datas, _i64([x for p in bot_phys for x in p]), int(r0),
                                                  int(r1)))
    return float(dd[0])
