#!/usr/bin/env python
"""bench.py — einsumsvd throughput on BASELINE config 2 (the metric's headline config).

Workload: one standalone two-layer row absorb,
``two_layer_apply_row`` on a length-8 boundary MPS with m = 64 (N(0,1) entries)
absorbing one interior double-layer row of r = 8, d = 2 sites (bra = ket,
N(0,1)), truncated back to m = 64 by implicit randomized SVD with oversample 8
(k = 72) and 2 power iterations; sketch seeded as the reference does
(derive_seed(seed, 0x20, row, col)).  One step = one row absorb = 7 einsumsvd.

metric/unit: BASELINE.json's metric as einsumsvd FP64 TFLOP/s = the row's
ALGORITHMIC real FP64 flops / time, counted the SURVEY §8(d) real-aware way:
the reference's own contraction order and instr::flops terms
(paper_2006_15234_b200/costmodel.py, pinned against the reference counter in
tests/test_costmodel.py), 8 real flops per complex multiply-add, 4 where one
operand is a real PEPS site (the BASELINE PEPS are real).  2.067e12 flops per
config-2 row.  The reference-counter rate (4 x instr::flops = 2.750e12 per row,
every product counted complex) is reported beside it as
``value_reference_counter``.  ms_per_step is the seconds-per-row-absorb figure.
Inputs (611 MB of intermediates per apply) exceed the 126 MB L2, so no explicit
flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference: the compiled reference (oracle/_ref: the unmodified
reference sources + OpenBLAS, all host threads) on rank 0; each step is one
ImplicitOperator::apply + adjoint_apply (implicit.cpp:66-100) at the config-2
interior-column size (the operator applications are 84 % of an einsumsvd's
flops; a whole column takes ~27 s on 16 cores, so K = 20 columns would not fit
"a few minutes"); rate = the same real-aware flop count of those two calls /
their time.

N > 1 (torchrun): ONE config-2 row absorb split across the N ranks along the
boundary bond by the C++ bond-sharded driver behind the C ABI (NCCL on the
library stream), scaling "strong", value = the row's flops / the
max over ranks of the device time; --replicas runs N independent rows instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from paper_2006_15234_b200 import costmodel, inputs  # noqa: E402

METRIC = "PEPS boundary-contraction s/norm; einsumsvd FP64 TFLOP/s & % of DMMA peak"
UNIT = "TFLOP/s"
L, R, M, Q, OS = 8, 8, 64, 2, 8
COLUMN_LABELS = ["apqsmn", "uvst", "dumbe", "dvncf"]
COLUMN_SHAPES = [(M, R, R, M, R, R), (R, R, M, M), (2, R, R, R, R), (2, R, R, R, R)]
COLUMN_REAL = [False, False, True, True]  # pending v, top site S complex; bra/ket real


def workload_config(world=1):
    """Identical in both arms (the driver compares them)."""
    return {"workload": "config2: two_layer_apply_row, boundary L=8 m=64, PEPS row r=8 d=2, implicit rSVD k=72 q=2",
            "length": L, "bond_r": R, "boundary_m": M, "oversample": OS, "power_iters": Q, "probe_k": M + OS,
            "data_layout": "complex128 row-major (reference Tensor layout)",
            "l2": "inputs+intermediates (>600 MB per apply) exceed the 126 MB L2; no flush needed",
            "flop_count": "real-aware algorithmic (SURVEY 8(d)): 8 real flops per complex MAC, 4 with a real "
                          "PEPS-site operand; reference contraction order",
            "parallelism": f"replicas x{world}"}


def alg_flops_row():
    """Real-aware algorithmic real flops of one config-2 row absorb (2.067e12)."""
    return 4 * costmodel.two_layer_row_flops(L, R, M, Q, OS, real_sites=True)


def refcounter_flops_row():
    """4 x the reference's instr::flops of one config-2 row absorb (2.750e12)."""
    return 4 * costmodel.two_layer_row_flops(L, R, M, Q, OS)


def apply_pair_flops():
    """Real-aware real flops of one apply + one adjoint_apply at the config-2 column size."""
    k = M + OS
    cols = [R, R, M, R, R]  # b c t e f
    rows = [M, R, R]  # a p q
    rf = COLUMN_REAL + [False]
    ap = costmodel.network_flops(COLUMN_SHAPES + [cols + [k]], COLUMN_LABELS + ["bctefX"], "apqX", rf)
    ad = costmodel.network_flops(COLUMN_SHAPES + [rows + [k]], COLUMN_LABELS + ["apqX"], "bctefX", rf)
    return 4 * (ap + ad)


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- reference CPU samples

def _column_inputs(seed):
    """One interior column of config 2 (contraction.cpp:293-299), N(0,1) entries."""
    v = inputs.gaussian(COLUMN_SHAPES[0], seed)
    s = inputs.gaussian(COLUMN_SHAPES[1], seed + 1)
    b = inputs.gaussian(COLUMN_SHAPES[2], seed + 2)
    return [v, s, b.conj(), b]


class ApplyPairSample:
    """The reference arm's step: ImplicitOperator::apply(Omega) + adjoint_apply(P)
    (implicit.cpp:66-100) of one config-2 interior column on oracle/_ref, timed
    inside the reference (operator construction / marshalling excluded)."""

    def __init__(self, threads, seed=42):
        from oracle import ref  # bench's CPU-baseline leg only
        self.ref = ref
        ref.set_threads(threads)
        self.ts = _column_inputs(seed)
        k = M + OS
        self.omega = ref.random_tensor((R, R, M, R, R, k), inputs.derive_seed(seed, 0x20, 1, 3))
        self.p = ref.random_tensor((M, R, R, k), seed + 7)
        self.flops = apply_pair_flops()

    def step(self):
        _, ta = self.ref.implicit_apply(self.ts, COLUMN_LABELS, "apq", "bctef", self.omega, timed=True)
        _, tb = self.ref.implicit_apply(self.ts, COLUMN_LABELS, "apq", "bctef", self.p, adjoint=True, timed=True)
        return ta + tb


APPLY_PAIR_NOTE = ("one ImplicitOperator::apply + adjoint_apply of a config-2 interior column (v 64x8x8x64x8x8, "
                   "probe k=72) per step on oracle/_ref (unmodified reference sources, OpenBLAS 0.3.15), timed "
                   "inside the reference; the same real-aware flop count as the GPU arm")


def cpu_config_baselines(cores):
    """Per-config reference CPU timings on this box's host cores (bounded samples).

    config 1: mean of 10 full norms; config 3: one interior row absorb at the
    config-3 shapes (L=16, r=6, m=36, k=41), x15 rows for a norm; config 4: 10
    ITE steps from |+>; config 5: one interior column einsumsvd at m=64 r=8
    (the config-5 column), x31 columns x31 rows for a norm."""
    from oracle import ref
    ref.set_threads(cores)
    out = {"cores": cores, "kind": "reference"}
    c1 = inputs.config1()
    ref.contract_two_layer(c1["sites"], 4, 4, 4, c1["seed"], 1, 4)
    t0 = time.perf_counter()
    for _ in range(10):
        ref.contract_two_layer(c1["sites"], 4, 4, 4, c1["seed"], 1, 4)
    out["config1_s_per_norm"] = (time.perf_counter() - t0) / 10
    sites3, top3, phys3 = _row_inputs(16, 6, 36, 3)
    t0 = time.perf_counter()
    ref.two_layer_apply_row(top3, phys3, sites3, 3, 16, 1, 36, 3, 2, -1, True, 0x20)
    row3 = time.perf_counter() - t0
    out["config3_s_per_row_absorb"] = row3
    out["config3_s_per_norm_extrapolated"] = 15 * row3
    plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
    _, dt4 = ref.ite_tfim(plus, 8, 8, 1.0, 3.0, 0.01, 10, 8)
    out["config4_s_per_step"] = dt4 / 10
    ts = _column_inputs(42)
    r5 = ref.einsumsvd(ts, COLUMN_LABELS, "apq", "bctef", M, 1e-14, "implicit_rsvd", "right", Q, OS,
                       inputs.derive_seed(42, 0x20, 1, 3))
    out["config5_s_per_column"] = r5["seconds"]
    out["config5_s_per_norm_extrapolated"] = 31 * 31 * r5["seconds"]
    out["sample"] = ("config 1: mean of 10 norms; config 3: one interior row absorb (L=16 r=6 m=36) x 15 rows; "
                     "config 4: 10 ITE steps; config 5: one interior m=64 r=8 column einsumsvd x 31 x 31")
    return out


def _row_inputs(length, bond, m, seed):
    """A 3-row PEPS with the config's entry scaling and a Gaussian top boundary
    (bonds m): the inputs of one interior row absorb at that config's shapes."""
    scale = 1.0 / np.sqrt(bond * bond * 2)
    sites = inputs.random_peps(3, length, bond, seed, scale=scale)
    top, phys = inputs.random_boundary(length, (bond, bond), m, inputs.derive_seed(seed, 0x70), scale=0.1)
    return sites, top, phys


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    sample = ApplyPairSample(cores)
    for _ in range(max(0, args.warmup)):
        sample.step()
    times = [sample.step() for _ in range(args.steps)]
    per = statistics.median(times)
    value = sample.flops / per / 1e12
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded N(0,1) Box-Muller over SplitMix64)",
            "config": workload_config(world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": APPLY_PAIR_NOTE},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "sample_flops_per_step": sample.flops, "mean_ms_per_step": 1e3 * sum(times) / len(times)}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm

def run_b200(args, rank, world, local_rank):
    import torch
    import paper_2006_15234_b200.api as A

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
    ctx = A.Context(local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local_rank))

    c2 = inputs.config2(seed=2 + rank)
    host_sites = c2["sites"]
    host_top = c2["top"]
    st = A.PepsState(3, L, 2, host_sites, ctx=ctx)
    top = A.TwoLayerBoundary.from_sites(host_top, c2["phys"], ctx=ctx)
    opt = A.ContractOption.two_layer_opt(M, c2["seed"], Q, OS)

    for _ in range(max(args.warmup, 0)):
        out = A.two_layer_apply_row(top, st, st, 1, opt, 0x20)
    ctx.sync()
    del out

    # ---- timed region: device-resident inputs
    if dist:
        dist.barrier()
    ctx.sync()
    torch.cuda.synchronize()
    ctx.reset_counters()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            out = A.two_layer_apply_row(top, st, st, 1, opt, 0x20)
        e1.record(stream)
        ctx.sync()
        torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / args.steps
    launches = ctx.counters()["launches"]
    if dist:
        dist.barrier()
    del out

    # ---- e2e: public API with host buffers (pinned), H2D inputs + D2H result every step
    pinned_sites = [torch.from_numpy(s.view(np.float64)).pin_memory() for s in host_sites]
    pinned_top = [torch.from_numpy(s.view(np.float64)).pin_memory() for s in host_top]
    h2d = sum(s.nbytes for s in host_sites) + sum(s.nbytes for s in host_top)
    out_shapes = [(R * R, 1 if c == 0 else M, 1 if c == L - 1 else M) for c in range(L)]
    pinned_out = [torch.empty(int(np.prod(s)) * 2, dtype=torch.float64).pin_memory() for s in out_shapes]
    d2h = sum(p.numel() * 8 for p in pinned_out)

    def e2e_step():
        sites = [A.DeviceTensor(_from_pinned(ctx, p, s.shape), ctx) for p, s in zip(pinned_sites, host_sites)]
        tops = [A.DeviceTensor(_from_pinned(ctx, p, s.shape), ctx) for p, s in zip(pinned_top, host_top)]
        s2 = A.PepsState(3, L, 2, sites, ctx=ctx)
        t2 = A.TwoLayerBoundary.from_sites(tops, c2["phys"], ctx=ctx)
        o = A.two_layer_apply_row(t2, s2, s2, 1, opt, 0x20)
        for i, site in enumerate(o.sites):
            _to_pinned(ctx, site, pinned_out[i])
        ctx.sync()

    e2e_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    torch.cuda.synchronize()
    dt_e2e = (time.perf_counter() - t0) / args.steps

    # ---- roofline pass (instrumented, separate from the timed region).  The
    # eigensolver/GEMM overlap is switched off here so that every kernel's
    # event-timed duration is its own (two-stream concurrency would inflate both).
    ctx.set_option("overlap", 0)
    ctx.profile(True)
    out = A.two_layer_apply_row(top, st, st, 1, opt, 0x20)
    rep = ctx.profile_report()
    ctx.profile(False)
    ctx.set_option("overlap", 1)
    del out
    # ---- stream timeline of one row as timed (overlap on): where the row waits
    ctx.profile(True)
    out = A.two_layer_apply_row(top, st, st, 1, opt, 0x20)
    timeline = _timeline_summary(ctx.profile_timeline())
    ctx.profile(False)
    del out

    if dist:
        t = torch.tensor([dt, dt_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt, dt_e2e = float(t[0]), float(t[1])

    extra_roofs = {}
    if world == 1 and not args.no_norms:
        extra_roofs = config_rooflines(A, ctx)

    if rank != 0:
        return 0
    flops = alg_flops_row()
    value = world * flops / dt / 1e12
    peak = _fp64_peak()
    g = rep["gemm"]
    # achieved = real flops the DMMAs execute (3M launches: 6 per complex MAC,
    # 4M launches: 8, complex x real: 4) / device time of the GEMM launches --
    # the tensor-pipe roofline (a hardware fraction, <= 1).
    achieved = g["exec_flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else None
    achieved_alg = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else None
    total_ms = sum(v["ms"] for v in rep.values())
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak["tflops"], "unit": "TFLOP/s",
            "frac": achieved / peak["tflops"] if achieved else None, "traffic": _ncu_traffic(),
            "kernel": "zgemm_cx_kernel (complex FP64 GEMM on DMMA.8x8x4: 3M/Gauss, 4M complex-fragment and "
                      "complex x real instantiations, all launches of the step)",
            "achieved_unit_note": "executed DMMA real flops / GEMM device time (serialised profile pass)",
            "achieved_reference_counter": achieved_alg,
            "kernel_share_of_step": g["ms"] / total_ms if total_ms else None,
            "eigensolver_share_of_step": rep["small"]["ms"] / total_ms if total_ms else None,
            "profile_pass": "serialised (overlap off); the timed step overlaps the k x k eigensolver with GEMMs",
            "launches_per_step": g["launches"], "avg_launch_ms": g["ms"] / max(1, g["launches"]),
            "reference_counter_flops_per_step": g["flops"], "executed_flops_per_step": g["exec_flops"],
            "peak_source": peak["source"],
            "whole_step_executed_frac": (g["exec_flops"] / dt / 1e12) / peak["tflops"],
            "whole_step_value_frac": value / world / peak["tflops"],
            "breakdown_ms": {k: round(v["ms"], 3) for k, v in rep.items()}}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded N(0,1) Box-Muller over SplitMix64)",
            "config": workload_config(world), "s_per_row_absorb": dt,
            "value_reference_counter": world * refcounter_flops_row() / dt / 1e12,
            "clocks": clk.summary(), "gpu_launches": launches,
            "e2e": {"value": world * flops / dt_e2e / 1e12, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "s_per_step": dt_e2e},
            "roofline": roof}
    line["timeline"] = timeline
    if extra_roofs:
        line["roofline_configs"] = extra_roofs
    if world == 1 and not args.no_norms:
        line["s_per_norm"] = norm_timings(A, ctx)
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        try:
            sample = ApplyPairSample(cores)
            sample.step()  # warm
            ts = [sample.step() for _ in range(2)]
            cv = sample.flops / min(ts) / 1e12
            line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": cores, "kind": "reference",
                                    "sample": APPLY_PAIR_NOTE + f" (best of 2: {min(ts):.2f} s)"}
            if not args.no_norms:
                line["cpu_baseline_configs"] = cpu_config_baselines(cores)
        except Exception as e:  # oracle missing on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": cores, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    return 0


def _union_ms(iv):
    tot, cs, ce = 0.0, None, None
    for a, b in sorted(iv):
        if cs is None or a > ce:
            if cs is not None:
                tot += ce - cs
            cs, ce = a, b
        else:
            ce = max(ce, b)
    return tot + (ce - cs if cs is not None else 0.0)


def _timeline_summary(tl):
    """Per-launch events on both streams of one row (tools/timeline.py): span,
    busy time per stream, time with no kernel running, and the main stream's
    (latency chain's) work that ran while the side stream was idle, by kind."""
    if not tl:
        return None
    main = [(s, e) for k, s, e, f, sd in tl if sd == 0]
    side = sorted((s, e) for k, s, e, f, sd in tl if sd == 1)
    span = max(e for _, _, e, _, _ in tl) - min(s for _, s, _, _, _ in tl)
    exposed = {}
    for k, s, e, f, sd in tl:
        if sd:
            continue
        ov = sum(max(0.0, min(e, b) - max(s, a)) for a, b in side if b > s and a < e)
        exposed[k] = round(exposed.get(k, 0.0) + (e - s) - ov, 3)
    return {"span_ms": round(span, 3), "busy_main_ms": round(_union_ms(main), 3),
            "busy_side_ms": round(_union_ms(side), 3), "idle_ms": round(span - _union_ms(main + side), 3),
            "main_exposed_ms_by_kind": exposed,
            "note": "per-launch CUDA events on the main / side stream of one row absorb, overlap on "
                    "(event overhead included)"}


def config_rooflines(A, ctx):
    """Roofline of one interior row absorb at the config-3 and config-5 shapes
    (serialised profile pass, overlap off): executed DMMA flops / GEMM device
    time against the FP64 peak, and the k x k eigensolver's share of the
    serialised kernel time (the latency chain of the row)."""
    peak = _fp64_peak()["tflops"]
    out = {}
    for name, (length, bond, m, os_) in {"config3_row_L16_r6_m36": (16, 6, 36, -1),
                                         "config5_row_L32_r8_m64": (32, 8, 64, 8)}.items():
        sites, top, phys = _row_inputs(length, bond, m, 11)
        st = A.PepsState(3, length, 2, sites, ctx=ctx)
        tb = A.TwoLayerBoundary.from_sites(top, phys, ctx=ctx)
        opt = A.ContractOption.two_layer_opt(m, 11, 2, os_)
        A.two_layer_apply_row(tb, st, st, 1, opt, 0x20)  # warm the plans / pools
        ctx.sync()
        t0 = time.perf_counter()
        A.two_layer_apply_row(tb, st, st, 1, opt, 0x20)
        ctx.sync()
        wall = time.perf_counter() - t0
        ctx.set_option("overlap", 0)
        ctx.profile(True)
        A.two_layer_apply_row(tb, st, st, 1, opt, 0x20)
        rep = ctx.profile_report()
        ctx.profile(False)
        ctx.set_option("overlap", 1)
        g = rep["gemm"]
        total = sum(v["ms"] for v in rep.values())
        ach = g["exec_flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else None
        out[name] = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                     "frac": ach / peak if ach else None, "s_per_row_absorb": wall,
                     "gemm_share": g["ms"] / total if total else None,
                     "eigensolver_share": rep["small"]["ms"] / total if total else None,
                     "breakdown_ms": {k: round(v["ms"], 3) for k, v in rep.items()}}
    return out


def norm_timings(A, ctx):
    """The metric's other half: seconds per <psi|psi> by two-layer boundary
    contraction (contract_two_layer) on BASELINE configs 1, 3 and 5 and seconds
    per ITE step of config 4, through the public API (wall clock around
    synchronised calls; inputs resident).  Config 1: mean of 10 after a warm-up;
    configs 3 and 5: median of 3 after a warm-up; config 4: 20 steps."""
    out = {}
    c1 = inputs.config1()
    st = A.PepsState(4, 4, 2, c1["sites"], ctx=ctx)
    o1 = A.ContractOption.two_layer_opt(4, c1["seed"], 1, 4)
    A.contract_two_layer(st, st, o1)
    t0 = time.perf_counter()
    for _ in range(10):
        A.contract_two_layer(st, st, o1)
    out["config1_4x4_r2_m4"] = (time.perf_counter() - t0) / 10
    for name, cfg, m, q, os_ in (("config3_16x16_r6_m36", inputs.config3(), 36, 2, -1),
                                 ("config5_32x32_r8_m64", inputs.config5(), 64, 2, 8)):
        n = cfg["rows"]
        st = A.PepsState(n, n, 2, cfg["sites"], ctx=ctx)
        opt = A.ContractOption.two_layer_opt(m, cfg["seed"], q, os_)
        A.contract_two_layer(st, st, opt)
        ts = []
        for _ in range(3):
            ctx.sync()
            t0 = time.perf_counter()
            A.contract_two_layer(st, st, opt)
            ts.append(time.perf_counter() - t0)
        out[name] = statistics.median(ts)
        out[name + "_all"] = ts
        del st
    # config 3's full workload: the cached environments (both sweeps) plus all
    # 256 <Z_i> (one expectation over 256 one-site terms with shared band
    # environments, observables.cpp:335-422)
    c3 = inputs.config3()
    st = A.PepsState(16, 16, 2, c3["sites"], ctx=ctx)
    z = np.diag([1.0, -1.0]).astype(np.complex128)
    terms = [A.LocalTerm(1.0, [(r, c)], z) for r in range(16) for c in range(16)]
    # allow_complex: at m = 36 the truncated environments leave an imaginary part
    # of ~1e-3 on the 256-term sum, which the reference's expectation() rejects
    # as non-Hermitian (observables.cpp:413-418); the timing is the same work
    eo = A.ExpectationOptions(A.ContractOption.two_layer_opt(36, c3["seed"], 2, -1), True, True, True)
    A.expectation(st, terms, eo)
    ts = []
    for _ in range(3):
        ctx.sync()
        t0 = time.perf_counter()
        A.expectation(st, terms, eo)
        ts.append(time.perf_counter() - t0)
    out["config3_cache_plus_256_z"] = statistics.median(ts)
    del st
    plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
    st = A.PepsState(8, 8, 2, plus, ctx=ctx)
    A.ite_tfim(st, 1.0, 3.0, 0.01, 2, 8)
    ctx.sync()
    t0 = time.perf_counter()
    A.ite_tfim(st, 1.0, 3.0, 0.01, 20, 8)
    ctx.sync()
    out["config4_ite_8x8_r8_s_per_step"] = (time.perf_counter() - t0) / 20
    out["note"] = ("seconds per norm (config 4: per Trotter step; config3_cache_plus_256_z: both cached sweeps + "
                   "all 256 <Z_i>); wall clock, synchronised, one B200")
    return out


def _from_pinned(ctx, pinned, shape):
    import ctypes as C
    from paper_2006_15234_b200._lib import check, lib
    shp = (C.c_int64 * len(shape))(*shape)
    h = C.c_void_p()
    check(lib().pepsb_tensor_from_host(ctx.h, len(shape), shp, C.c_void_p(pinned.data_ptr()), C.byref(h)))
    return h


def _to_pinned(ctx, dt, pinned):
    """Stream-ordered D2H of a result tensor into pinned host memory (C ABI)."""
    import ctypes as C
    from paper_2006_15234_b200._lib import check, lib
    check(lib().pepsb_tensor_to_host_async(ctx.h, dt.h, C.c_void_p(pinned.data_ptr())))


def _fp64_peak():
    p = os.path.join(HERE, "profiles", "fp64_peak.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"tflops": float(d["roofline_peak_tflops"]), "source": "measured (profiles/fp64_peak.json, "
                "DMMA issue ceiling on this pool's B200)"}
    except Exception:
        return {"tflops": 37.0, "source": "fallback 37 TF/s (FP64 DMMA, measured earlier)"}


def _ncu_traffic():
    p = os.path.join(HERE, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


def run_sharded(args, rank, world, local_rank):
    """N > 1 (default) or --sharded: ONE config-2 row absorb split across the N
    ranks along the boundary bond by the C++ driver behind the C ABI
    (pepsb_two_layer_apply_row_sharded, csrc/sharded.cpp: NCCL all-reduce /
    all-gather on the library stream); scaling "strong", value = the row's
    algorithmic flops / max-over-ranks device time.  Also times one sharded
    config-5 norm (32x32, r=8, m=64)."""
    import torch
    import torch.distributed as dist
    import paper_2006_15234_b200.api as A

    torch.cuda.set_device(local_rank)
    ctx = A.Context(local_rank)
    if world > 1:
        A.comm_init_from_torch(ctx)
    else:
        A.comm_init(ctx, A.comm_unique_id(), 0, 1)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local_rank))
    c2 = inputs.config2(seed=2)
    st = A.PepsState(3, L, 2, c2["sites"], ctx=ctx)
    top = A.TwoLayerBoundary.from_sites(c2["top"], c2["phys"], ctx=ctx)
    opt = A.ContractOption.two_layer_opt(M, c2["seed"], Q, OS)

    for _ in range(max(args.warmup, 0)):
        out = A.two_layer_apply_row_sharded(top, st, st, 1, opt, 0x20)
    ctx.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.reset_counters()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            out = A.two_layer_apply_row_sharded(top, st, st, 1, opt, 0x20)
        e1.record(stream)
        ctx.sync()
        torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / args.steps
    launches = ctx.counters()["launches"]
    del out

    # e2e: inputs from pinned host memory, boundary copied back every step
    host_sites, host_top = c2["sites"], c2["top"]
    pinned_sites = [torch.from_numpy(x.view(np.float64)).pin_memory() for x in host_sites]
    pinned_top = [torch.from_numpy(x.view(np.float64)).pin_memory() for x in host_top]
    h2d = sum(x.nbytes for x in host_sites) + sum(x.nbytes for x in host_top)
    out_shapes = [(R * R, 1 if c == 0 else M, 1 if c == L - 1 else M) for c in range(L)]
    pinned_out = [torch.empty(int(np.prod(x)) * 2, dtype=torch.float64).pin_memory() for x in out_shapes]
    d2h = sum(p.numel() * 8 for p in pinned_out)

    def e2e_step():
        sites = [A.DeviceTensor(_from_pinned(ctx, p, x.shape), ctx) for p, x in zip(pinned_sites, host_sites)]
        tops = [A.DeviceTensor(_from_pinned(ctx, p, x.shape), ctx) for p, x in zip(pinned_top, host_top)]
        s2 = A.PepsState(3, L, 2, sites, ctx=ctx)
        t2 = A.TwoLayerBoundary.from_sites(tops, c2["phys"], ctx=ctx)
        o = A.two_layer_apply_row_sharded(t2, s2, s2, 1, opt, 0x20)
        for i, site in enumerate(o.sites):
            _to_pinned(ctx, site, pinned_out[i])
        ctx.sync()

    e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    dt_e2e = (time.perf_counter() - t0) / args.steps

    norm5 = None
    if not args.no_norms:
        c5 = inputs.config5()
        st5 = A.PepsState(32, 32, 2, c5["sites"], ctx=ctx)
        opt5 = A.ContractOption.two_layer_opt(64, c5["seed"], 2, 8)
        if world > 1:
            dist.barrier()
        ctx.sync()
        t0 = time.perf_counter()
        A.contract_two_layer_sharded(st5, st5, opt5)
        ctx.sync()
        norm5 = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt, dt_e2e, norm5 or 0.0], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt, dt_e2e, norm5 = float(t[0]), float(t[1]), (float(t[2]) if norm5 is not None else None)
    A.comm_destroy(ctx)
    if rank != 0:
        return 0
    flops = alg_flops_row()
    line = {"metric": METRIC, "value": flops / dt / 1e12, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded N(0,1) Box-Muller over SplitMix64)",
            "config": dict(workload_config(world),
                           parallelism=f"bond-sharded x{world} (t / s of the boundary bond, NCCL)"),
            "s_per_row_absorb": dt,
            "value_reference_counter": refcounter_flops_row() / dt / 1e12,
            "clocks": clk.summary(), "gpu_launches": launches,
            "e2e": {"value": flops / dt_e2e / 1e12, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "s_per_step": dt_e2e}}
    if norm5 is not None:
        line["s_per_norm"] = {"config5_32x32_r8_m64_sharded": norm5,
                              "note": "one bond-sharded contract_two_layer on all ranks (max over ranks)"}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-norms", action="store_true", help="skip the per-config s/norm timings (configs 1, 3, 5, 4)")
    ap.add_argument("--sharded", action="store_true",
                    help="run the bond-sharded C++ driver even at N=1 (N>1 always does)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent single-GPU replicas (weak scaling) instead of the sharded row")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    try:
        if args.sharded or (world > 1 and not args.replicas):
            return run_sharded(args, rank, world, local_rank)
        return run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
