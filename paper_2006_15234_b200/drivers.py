"""Host-side drivers over the device library.

Mirrors the reference's orchestration layer, which is host code there too:

- gates / Observable text format / build_j1j2   observables.cpp:21-254, state.cpp:301-383
- energy_contract_option / state_energy         drivers.cpp:33-53
- nelder_mead / cobyla_lite / minimize          optimize.cpp:37-194
- run_vqe (+ theta0 initialisation)             drivers.cpp:134-191
- run_expect_json / run_vqe_json / run_ite_json drivers.cpp:265-550 (schema-1 result documents)

Every contraction, truncation and expectation value runs on the device
(paper_2006_15234_b200.api); only scalars and small gate matrices live on the
host.  Errors follow the reference family (ConfigError for bad configs, via
api.PepsError kinds).
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import api as A
from .api import LocalTerm, PepsError
from .inputs import derive_seed, splitmix_stream, unit

_CONFIG, _VALIDATION = 5, 2

# ----------------------------------------------------------------------------- gates (state.cpp:301-383)

X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
I2 = np.eye(2, dtype=np.complex128)
PAULIS = {"X": X, "Y": Y, "Z": Z, "I": I2}


def two_site(a, b) -> np.ndarray:
    """gates::two_site: a (x) b as (out, out, in, in)."""
    return np.einsum("ac,bd->abcd", np.asarray(a, dtype=np.complex128), np.asarray(b, dtype=np.complex128))


# ----------------------------------------------------------------------------- observables (observables.cpp)

def _check_one(op):
    op = np.asarray(op, dtype=np.complex128)
    if op.ndim != 2 or op.shape[0] != op.shape[1]:
        raise PepsError(1, "one-site term operator must be d x d")
    return op


def build_j1j2(rows: int, cols: int, j1=(1.0, 1.0, 1.0), j2=(0.0, 0.0, 0.0), h=(0.0, 0.0, 0.0)) -> List[LocalTerm]:
    """build_j1j2 (observables.cpp:61-96): fields, then J1 horizontal / vertical
    pairs, then J2 diagonals, Pauli X, Y, Z per coupling, zero couplings skipped."""
    if rows == 0 or cols == 0:
        raise PepsError(_VALIDATION, "grid must be non-empty")
    ps = [X, Y, Z]
    out: List[LocalTerm] = []
    for r in range(rows):
        for c in range(cols):
            for p in range(3):
                if h[p] != 0.0:
                    out.append(LocalTerm(h[p], [(r, c)], ps[p]))

    def pair(a, b, k):
        for p in range(3):
            if k[p] != 0.0:
                out.append(LocalTerm(k[p], [a, b], two_site(ps[p], ps[p])))

    for r in range(rows):
        for c in range(cols - 1):
            pair((r, c), (r, c + 1), j1)
    for r in range(rows - 1):
        for c in range(cols):
            pair((r, c), (r + 1, c), j1)
    for r in range(rows - 1):
        for c in range(cols):
            if c + 1 < cols:
                pair((r, c), (r + 1, c + 1), j2)
            if c > 0:
                pair((r, c), (r + 1, c - 1), j2)
    return out


def _parse_coeff(tok: str) -> complex:
    if tok.startswith("("):
        comma, close = tok.find(","), tok.find(")")
        if comma < 0 or close < 0:
            raise PepsError(_VALIDATION, f"bad complex coefficient '{tok}'")
        return complex(float(tok[1:comma]), float(tok[comma + 1:close]))
    return complex(float(tok), 0.0)


def _parse_site(tok: str, pos: int):
    if pos >= len(tok) or tok[pos] != "(":
        raise PepsError(_VALIDATION, f"expected '(' in '{tok}'")
    comma, close = tok.find(",", pos), tok.find(")", pos)
    if comma < 0 or close < 0:
        raise PepsError(_VALIDATION, f"bad site in '{tok}'")
    return (int(tok[pos + 1:comma]), int(tok[comma + 1:close])), close + 1


def _parse_op(tok: str):
    if len(tok) >= 2 and tok[0] in PAULIS and tok[1] == "@":
        site, _ = _parse_site(tok, 2)
        return PAULIS[tok[0]], site
    if tok.startswith("M["):
        close = tok.find("]")
        if close < 0:
            raise PepsError(_VALIDATION, f"unterminated matrix in '{tok}'")
        vals = []
        for item in tok[2:close].split(","):
            if ":" in item:
                re_, im = item.split(":", 1)
                vals.append(complex(float(re_), float(im)))
            else:
                vals.append(complex(float(item), 0.0))
        d = int(round(math.sqrt(len(vals))))
        if d * d != len(vals):
            raise PepsError(_VALIDATION, "matrix entry count must be a square")
        pos = close + 1
        if pos >= len(tok) or tok[pos] != "@":
            raise PepsError(_VALIDATION, f"expected '@' in '{tok}'")
        site, _ = _parse_site(tok, pos + 1)
        return np.array(vals, dtype=np.complex128).reshape(d, d), site
    raise PepsError(_VALIDATION, f"cannot parse operator token '{tok}'")


def observable_parse(text: str) -> List[LocalTerm]:
    """Observable::parse (observables.cpp:190-215): one term per line,
    'coeff OP@(r,c) [OP@(r,c)]' with OP a Pauli letter or M[...] (re[:im],...)."""
    out: List[LocalTerm] = []
    for line in text.splitlines():
        s = line.strip(" \t\r")
        if not s or s.lstrip(" \t").startswith("#"):
            continue
        toks = s.split()
        coeff = _parse_coeff(toks[0])
        ops = [_parse_op(t) for t in toks[1:]]
        if not ops or len(ops) > 2:
            raise PepsError(_VALIDATION, f"each term needs one or two operators: '{line}'")
        if len(ops) == 1:
            out.append(LocalTerm(coeff, [ops[0][1]], _check_one(ops[0][0])))
        else:
            if ops[0][1] == ops[1][1]:
                raise PepsError(_VALIDATION, "two-site term needs distinct sites")
            out.append(LocalTerm(coeff, [ops[0][1], ops[1][1]], two_site(ops[0][0], ops[1][0])))
    return out


def hamiltonian_from_json(j, rows: int, cols: int) -> List[LocalTerm]:
    """drivers.cpp:289-305: {"type": "j1j2", "j1", "j2", "h"} or {"type": "text", "terms"}."""
    if not isinstance(j, dict):
        raise PepsError(_CONFIG, "hamiltonian must be an object")
    typ = j.get("type", "j1j2")
    if typ == "j1j2":
        def triple(key, fallback):
            if key not in j:
                return (fallback,) * 3
            v = j[key]
            if isinstance(v, (int, float)) and not isinstance(v, bool):
                return (float(v),) * 3
            if isinstance(v, list) and len(v) == 3:
                return tuple(float(x) for x in v)
            raise PepsError(_CONFIG, f"hamiltonian.{key} must be a number or [x,y,z]")
        return build_j1j2(rows, cols, triple("j1", 1.0), triple("j2", 0.0), triple("h", 0.0))
    if typ == "text":
        if "terms" not in j:
            raise PepsError(_CONFIG, "hamiltonian.terms missing")
        return observable_parse(j["terms"])
    raise PepsError(_CONFIG, f"unknown hamiltonian type '{typ}'")


# ----------------------------------------------------------------------------- energies (drivers.cpp:33-53)

FAMILIES = ("exact", "bmps", "ibmps", "two-layer-ibmps")


def energy_contract_option(family: str, m: int, rsvd_iters: int, seed: int) -> A.ContractOption:
    """drivers.cpp:33-44: exact SVD truncation for the exact / bmps families,
    implicit randomized SVD otherwise (the expectation always runs the
    two-layer cached sweeps, observables.cpp:348-360)."""
    if family not in FAMILIES:
        raise PepsError(_CONFIG, f"unknown contraction family '{family}'")
    strategy = A.SvdStrategy.exact if family in ("exact", "bmps") else A.SvdStrategy.implicit_rsvd
    return A.ContractOption(A.TruncationPolicy(m, 1e-14), strategy, A.RsvdConfig(rsvd_iters, -1, 0), True, seed)


def state_energy(s: A.PepsState, terms, family: str, m: int, rsvd_iters: int, seed: int) -> float:
    """drivers.cpp:46-53: cached, shared environments."""
    opt = A.ExpectationOptions(energy_contract_option(family, m, rsvd_iters, seed), True, True, False)
    return A.expectation(s, terms, opt).value


# ----------------------------------------------------------------------------- optimizers (optimize.cpp)

@dataclass
class OptimConfig:
    max_evaluations: int = 300
    tolerance: float = 1e-6
    initial_step: float = 0.4


@dataclass
class OptimResult:
    best_f: float = 0.0
    best_x: List[float] = field(default_factory=list)
    trace: List[float] = field(default_factory=list)
    evaluations: int = 0
    status: str = "max-evaluations"


class _Budget(Exception):
    pass


class _Tracker:
    """optimize.cpp:14-33: counts evaluations, keeps the trace and the best point."""

    def __init__(self, f, res: OptimResult, budget: int):
        self.f, self.res, self.budget = f, res, budget

    def __call__(self, x) -> float:
        if self.res.evaluations >= self.budget:
            raise _Budget()
        v = float(self.f(list(x)))
        self.res.evaluations += 1
        self.res.trace.append(v)
        if len(self.res.trace) == 1 or v < self.res.best_f:
            self.res.best_f = v
            self.res.best_x = list(x)
        return v


def nelder_mead(f: Callable, x0: Sequence[float], cfg: OptimConfig) -> OptimResult:
    """optimize.cpp:37-115 (reflection -1, expansion -2, contractions -0.5 / 0.5, shrink 0.5)."""
    n = len(x0)
    res = OptimResult()
    ev = _Tracker(f, res, cfg.max_evaluations)
    pts = [list(map(float, x0)) for _ in range(n + 1)]
    fv = [0.0] * (n + 1)
    try:
        for i in range(1, n + 1):
            pts[i][i - 1] += cfg.initial_step
        for i in range(n + 1):
            fv[i] = ev(pts[i])
        while True:
            order = sorted(range(n + 1), key=lambda i: fv[i])  # stable, as std::sort on distinct keys
            pts = [pts[i] for i in order]
            fv = [fv[i] for i in order]
            if abs(fv[n] - fv[0]) < cfg.tolerance * (abs(fv[0]) + cfg.tolerance):
                res.status = "converged"
                break
            centroid = [0.0] * n
            for i in range(n):
                for j in range(n):
                    centroid[j] += pts[i][j] / float(n)

            def blend(t):
                return [centroid[j] + t * (pts[n][j] - centroid[j]) for j in range(n)]

            xr = blend(-1.0)
            fr = ev(xr)
            if fr < fv[0]:
                xe = blend(-2.0)
                fe = ev(xe)
                if fe < fr:
                    pts[n], fv[n] = xe, fe
                else:
                    pts[n], fv[n] = xr, fr
            elif fr < fv[n - 1]:
                pts[n], fv[n] = xr, fr
            else:
                xc = blend(-0.5 if fr < fv[n] else 0.5)
                fc = ev(xc)
                if fc < min(fr, fv[n]):
                    pts[n], fv[n] = xc, fc
                else:
                    for i in range(1, n + 1):
                        pts[i] = [pts[0][j] + 0.5 * (pts[i][j] - pts[0][j]) for j in range(n)]
                        fv[i] = ev(pts[i])
    except _Budget:
        pass
    return res


def cobyla_lite(f: Callable, x0: Sequence[float], cfg: OptimConfig) -> OptimResult:
    """optimize.cpp:117-187: linear model from the simplex edges (LU solve), a
    step of length rho down the model gradient, rho halved on failure."""
    n = len(x0)
    res = OptimResult()
    ev = _Tracker(f, res, cfg.max_evaluations)
    rho = cfg.initial_step
    rho_end = max(cfg.tolerance, 1e-10)
    pts = [list(map(float, x0)) for _ in range(n + 1)]
    fv = [0.0] * (n + 1)
    try:
        for i in range(1, n + 1):
            pts[i][i - 1] += rho
        for i in range(n + 1):
            fv[i] = ev(pts[i])
        while rho > rho_end:
            best = 0
            for i in range(1, n + 1):
                if fv[i] < fv[best]:
                    best = i
            pts[0], pts[best] = pts[best], pts[0]
            fv[0], fv[best] = fv[best], fv[0]
            a = np.array([[pts[i + 1][j] - pts[0][j] for j in range(n)] for i in range(n)], dtype=np.float64)
            g = np.array([fv[i + 1] - fv[0] for i in range(n)], dtype=np.float64)
            try:
                g = np.linalg.solve(a, g)  # dgesv: LU with partial pivoting
                singular = False
            except np.linalg.LinAlgError:
                singular = True
            if singular:
                for i in range(1, n + 1):
                    pts[i] = list(pts[0])
                    pts[i][i - 1] += rho
                    fv[i] = ev(pts[i])
                continue
            gnorm = math.sqrt(float(np.dot(g, g)))
            if gnorm < 1e-14:
                rho *= 0.5
                continue
            xt = [pts[0][j] - rho * g[j] / gnorm for j in range(n)]
            ft = ev(xt)
            if ft < fv[0]:
                worst = 0
                for i in range(1, n + 1):
                    if fv[i] > fv[worst]:
                        worst = i
                pts[worst], fv[worst] = xt, ft
            else:
                rho *= 0.5
                for i in range(1, n + 1):
                    pts[i] = [pts[0][j] + 0.5 * (pts[i][j] - pts[0][j]) for j in range(n)]
                    fv[i] = ev(pts[i])
        res.status = "converged"
    except _Budget:
        pass
    return res


def minimize(method: str, f: Callable, x0: Sequence[float], cfg: OptimConfig) -> OptimResult:
    """optimize.cpp:189-194."""
    if method == "nelder-mead":
        return nelder_mead(f, x0, cfg)
    if method == "cobyla":
        return cobyla_lite(f, x0, cfg)
    raise PepsError(_CONFIG, f"unknown optimizer '{method}' (use nelder-mead or cobyla)")


# ----------------------------------------------------------------------------- VQE (drivers.cpp:100-191)

@dataclass
class VqeConfig:
    """drivers.hpp:37-53."""
    rows: int = 4
    cols: int = 4
    hamiltonian: List[LocalTerm] = field(default_factory=list)
    layers: int = 2
    theta0: List[float] = field(default_factory=list)
    init: str = "random"
    optimizer: str = "nelder-mead"
    max_evaluations: int = 300
    tolerance: float = 1e-6
    initial_step: float = 0.4
    evolution_rank: int = 2
    contraction_rank: int = 16
    family: str = "two-layer-ibmps"
    rsvd_iters: int = 1
    update: str = "qr-svd-gram"
    seed: int = 0


@dataclass
class VqeOutcome:
    best_energy: float
    best_theta: List[float]
    trace: List[float]
    running_minimum: List[float]
    evaluations: int


class _SplitMix:
    """SplitMix64 (rng.hpp:12-32): next_symmetric = 2 * next_unit - 1."""

    def __init__(self, seed: int):
        self.seed, self.i = seed, 0

    def next_symmetric(self) -> float:
        u = unit(splitmix_stream(self.seed, 1, self.i))[0]
        self.i += 1
        return 2.0 * float(u) - 1.0


def _check_update(update: str):
    if update != "qr-svd-gram":
        if update in ("direct", "qr-svd"):
            raise PepsError(_CONFIG, f"update strategy '{update}' is not on the device path (use qr-svd-gram)")
        raise PepsError(_CONFIG, f"unknown update strategy '{update}'")


def run_vqe(cfg: VqeConfig, ctx: Optional[A.Context] = None) -> VqeOutcome:
    """run_vqe (drivers.cpp:134-191): seeded theta0 (random: pi * U[-1,1]; neel:
    pi on the odd checkerboard of layer 0 + 0.2 U[-1,1]), then the optimizer on
    theta -> state_energy(vqe_ansatz_state(theta)) seeded derive_seed(seed, 0xF)."""
    _check_update(cfg.update)
    n_params = cfg.layers * cfg.rows * cfg.cols
    theta0 = list(cfg.theta0)
    if not theta0:
        theta0 = [0.0] * n_params
        gen = _SplitMix(derive_seed(cfg.seed, 0x7E))
        if cfg.init == "random":
            theta0 = [math.pi * gen.next_symmetric() for _ in range(n_params)]
        elif cfg.init == "neel":
            for layer in range(cfg.layers):
                for r in range(cfg.rows):
                    for c in range(cfg.cols):
                        base = math.pi if (layer == 0 and (r + c) % 2 == 1) else 0.0
                        theta0[layer * cfg.rows * cfg.cols + r * cfg.cols + c] = base + 0.2 * gen.next_symmetric()
        else:
            raise PepsError(_CONFIG, f"unknown vqe init '{cfg.init}' (use random or neel)")
    if len(theta0) != n_params:
        raise PepsError(_CONFIG, "theta length must be layers * rows * cols")
    es = derive_seed(cfg.seed, 0xF)
    if cfg.layers == 0:
        st = A.computational_basis(cfg.rows, cfg.cols, [0] * (cfg.rows * cfg.cols), ctx=ctx)
        e = state_energy(st, cfg.hamiltonian, cfg.family, cfg.contraction_rank, cfg.rsvd_iters, es)
        return VqeOutcome(e, [], [e], [e], 1)

    def objective(theta):
        st = A.vqe_ansatz_state(cfg.rows, cfg.cols, cfg.layers, theta, cfg.evolution_rank, ctx)
        return state_energy(st, cfg.hamiltonian, cfg.family, cfg.contraction_rank, cfg.rsvd_iters, es)

    r = minimize(cfg.optimizer, objective, theta0,
                 OptimConfig(cfg.max_evaluations, cfg.tolerance, cfg.initial_step))
    running, rm = (r.trace[0] if r.trace else 0.0), []
    for v in r.trace:
        running = min(running, v)
        rm.append(running)
    return VqeOutcome(r.best_f, r.best_x, r.trace, rm, r.evaluations)


# ----------------------------------------------------------------------------- JSON front ends (drivers.cpp:265-550)

def _parse_config(text: str) -> dict:
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise PepsError(_CONFIG, f"config JSON parse error at line {e.lineno}, column {e.colno}: {e.msg}")
    if not isinstance(j, dict) or not isinstance(j.get("schema"), int) or isinstance(j.get("schema"), bool) \
            or j["schema"] != 1:
        raise PepsError(_CONFIG, 'config must declare "schema": 1')
    return j


def _skeleton(command: str, cfg: dict) -> dict:
    """drivers.cpp:322-331."""
    return {"schema": 1, "command": command, "config": cfg, "results": {}, "instrumentation": [],
            "versions": {"peps2d": "1.0.0", "result_format": 1}}


def run_expect_json(config_json: str, ctx: Optional[A.Context] = None) -> str:
    """run_expect_json (drivers.cpp:509-550): load the PEPS container named by
    "state", build the observable ("hamiltonian" or "observable_file"), run the
    device expectation with energy_contract_option(family, m, rsvd_iters, seed)
    and emit the reference's result document."""
    t0 = time.perf_counter()
    j = _parse_config(config_json)
    if "state" not in j:
        raise PepsError(_CONFIG, "expect config needs a state file path")
    st = A.load_peps(str(j["state"]), ctx=ctx)
    if "hamiltonian" in j:
        terms = hamiltonian_from_json(j["hamiltonian"], st.rows, st.cols)
    elif "observable_file" in j:
        try:
            with open(j["observable_file"]) as f:
                text = f.read()
        except OSError:
            raise PepsError(_CONFIG, "cannot open observable file")
        terms = observable_parse(text)
    else:
        raise PepsError(_CONFIG, "expect config needs hamiltonian or observable_file")
    opt = A.ExpectationOptions(energy_contract_option(j.get("family", "two-layer-ibmps"), int(j.get("m", 16)),
                                                      int(j.get("rsvd_iters", 1)), int(j.get("seed", 0))),
                               bool(j.get("use_cache", True)), bool(j.get("shared_environments", False)), False)
    r = A.expectation(st, terms, opt)
    doc = _skeleton("expect", j)
    doc["results"] = {"value": r.value, "value_per_site": r.value / (st.rows * st.cols),
                      "raw_sum_re": r.raw_sum.real, "raw_sum_im": r.raw_sum.imag, "norm_sq": r.norm_sq,
                      "full_sweeps": r.full_sweeps, "band_contractions": r.band_contractions, "flops": r.flops}
    doc["timing"] = {"seconds": time.perf_counter() - t0}
    return json.dumps(doc, indent=2)


def run_vqe_json(config_json: str, ctx: Optional[A.Context] = None) -> str:
    """run_vqe_json (drivers.cpp:384-425)."""
    t0 = time.perf_counter()
    j = _parse_config(config_json)
    cfg = VqeConfig(rows=int(j.get("rows", 4)), cols=int(j.get("cols", 4)), layers=int(j.get("layers", 2)))
    if "theta0" in j:
        cfg.theta0 = [float(x) for x in j["theta0"]]
    cfg.init = j.get("init", "random")
    if "optimizer" in j:
        o = j["optimizer"]
        cfg.optimizer = o.get("name", "nelder-mead")
        cfg.max_evaluations = int(o.get("max_evaluations", 300))
        cfg.tolerance = float(o.get("tolerance", 1e-6))
        cfg.initial_step = float(o.get("initial_step", 0.4))
    cfg.evolution_rank = int(j.get("evolution_rank", 2))
    cfg.contraction_rank = int(j.get("contraction_rank", 16))
    cfg.family = j.get("family", "two-layer-ibmps")
    if cfg.family not in FAMILIES:
        raise PepsError(_CONFIG, f"unknown contraction family '{cfg.family}'")
    cfg.rsvd_iters = int(j.get("rsvd_iters", 1))
    cfg.update = j.get("update", "qr-svd-gram")
    cfg.seed = int(j.get("seed", 0))
    if "hamiltonian" not in j:
        raise PepsError(_CONFIG, "vqe config needs a hamiltonian")
    cfg.hamiltonian = hamiltonian_from_json(j["hamiltonian"], cfg.rows, cfg.cols)
    out = run_vqe(cfg, ctx)
    doc = _skeleton("vqe", j)
    doc["results"] = {"best_energy": out.best_energy, "best_energy_per_site": out.best_energy / (cfg.rows * cfg.cols),
                      "best_theta": out.best_theta, "evaluations": out.evaluations, "trace": out.trace,
                      "running_minimum": out.running_minimum}
    doc["timing"] = {"seconds": time.perf_counter() - t0}
    return json.dumps(doc, indent=2)


def run_ite_json(config_json: str, ctx: Optional[A.Context] = None) -> str:
    """run_ite_json (drivers.cpp:335-382) over api.run_ite."""
    t0 = time.perf_counter()
    j = _parse_config(config_json)
    rows, cols = int(j.get("rows", 4)), int(j.get("cols", 4))
    family = j.get("family", "two-layer-ibmps")
    if family != "two-layer-ibmps":
        raise PepsError(_CONFIG, f"run_ite on the device supports family two-layer-ibmps (got '{family}')")
    _check_update(j.get("update", "qr-svd-gram"))
    if "hamiltonian" not in j:
        raise PepsError(_CONFIG, "ite config needs a hamiltonian")
    terms = hamiltonian_from_json(j["hamiltonian"], rows, cols)
    energies, st = A.run_ite(rows, cols, terms, float(j.get("tau", 0.02)), int(j.get("steps", 150)),
                             int(j.get("evolution_rank", 2)), int(j.get("contraction_rank", 4)),
                             int(j.get("rsvd_iters", 1)), int(j.get("energy_every", 1)), j.get("initial", "neel"),
                             int(j.get("seed", 0)), ctx=ctx)
    doc = _skeleton("ite", j)
    max_bond = max(max(s.shape[1:]) for s in st.sites)
    doc["results"] = {"energies": [{"step": s, "energy": e, "energy_per_site": e / (rows * cols)}
                                   for s, e in energies],
                      "final_energy": energies[-1][1] if energies else 0.0, "final_max_bond": int(max_bond)}
    doc["timing"] = {"seconds": time.perf_counter() - t0}
    return json.dumps(doc, indent=2)
