#!/usr/bin/env python
"""bench.py — einsumsvd throughput on BASELINE config 2 (the metric's headline config).

Workload: one standalone two-layer row absorb,
``two_layer_apply_row`` on a length-8 boundary MPS with m = 64 (N(0,1) entries)
absorbing one interior double-layer row of r = 8, d = 2 sites (bra = ket,
N(0,1)), truncated back to m = 64 by implicit randomized SVD with oversample 8
(k = 72) and 2 power iterations; sketch seeded as the reference does
(derive_seed(seed, 0x20, row, col)).  One step = one row absorb = 7 einsumsvd.

metric/unit: BASELINE.json's metric, reported as einsumsvd FP64 TFLOP/s =
4 x (the reference's own instr::flops count of the row absorb, reproduced
exactly by paper_2006_15234_b200/costmodel.py and pinned against the oracle in
tests/test_costmodel.py) / time.  ms_per_step is the seconds-per-row-absorb
figure.  Inputs (611 MB of intermediates per apply) exceed the 126 MB L2, so no
explicit flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 (torchrun): the row-absorb chain is sequential, so ranks run
independent replicas (scaling "weak"); value = sum of all ranks' work / max
over ranks of the device time.
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


def workload_config(extra=None):
    cfg = {"workload": "config2: two_layer_apply_row, boundary L=8 m=64, PEPS row r=8 d=2, implicit rSVD k=72 q=2",
           "length": L, "bond_r": R, "boundary_m": M, "oversample": OS, "power_iters": Q, "probe_k": M + OS,
           "data_layout": "complex128 row-major (reference Tensor layout)",
           "l2": "inputs+intermediates (>600 MB per apply) exceed the 126 MB L2; no flush needed",
           "parallelism": "replicas"}
    if extra:
        cfg.update(extra)
    return cfg


def alg_flops_row():
    return 4 * costmodel.two_layer_row_flops(L, R, M, Q, OS)


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


# ----------------------------------------------------------------------------- reference CPU sample

def cpu_sample(threads: int, seed: int = 42):
    """One interior-column einsumsvd of config 2 on the compiled reference (oracle/_ref).

    Pending tensor v (a,p,q,s,m,n) = (64,8,8,64,8,8), top site (8,8,64,64), bra/ket
    (2,8,8,8,8): exactly the interior-column network of two_layer_apply_row
    (contraction.cpp:293-299), N(0,1) entries.  Returns (seconds, algorithmic real flops).
    """
    from oracle import ref  # bench's CPU-baseline leg only
    ref.set_threads(threads)
    v = inputs.gaussian((M, R, R, M, R, R), seed)
    s = inputs.gaussian((R, R, M, M), seed + 1)
    b = inputs.gaussian((2, R, R, R, R), seed + 2)
    ts = [v, s, b.conj(), b]
    labels = ["apqsmn", "uvst", "dumbe", "dvncf"]
    t0 = time.perf_counter()
    ref.einsumsvd(ts, labels, "apq", "bctef", M, 1e-14, "implicit_rsvd", "right", Q, OS,
                  inputs.derive_seed(seed, 0x20, 1, 3))
    dt = time.perf_counter() - t0
    fl = 4 * costmodel.rsvd_flops([t.shape for t in ts], labels, "apq", "bctef", M, Q, OS)
    return dt, fl


def cpu_sample_small(threads: int):
    from oracle import ref
    ref.set_threads(threads)
    v = inputs.gaussian((16, 4, 4, 16, 4, 4), 1)
    s = inputs.gaussian((4, 4, 16, 16), 2)
    b = inputs.gaussian((2, 4, 4, 4, 4), 3)
    ref.einsumsvd([v, s, b.conj(), b], ["apqsmn", "uvst", "dumbe", "dvncf"], "apq", "bctef", 16, 1e-14,
                  "implicit_rsvd", "right", Q, OS, 7)


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    for _ in range(max(0, args.warmup)):
        cpu_sample_small(cores)
    budget = float(os.environ.get("PEPSB_REF_BUDGET_S", "150"))
    times, flops = [], 0.0
    t_start = time.perf_counter()
    for i in range(args.steps):
        dt, fl = cpu_sample(cores, seed=42 + i)
        times.append(dt)
        flops = fl
        if time.perf_counter() - t_start > budget:
            break
    per = statistics.median(times)
    value = flops / per / 1e12
    sample = ("one interior-column einsumsvd of config 2 (v 64x8x8x64x8x8, k=72, q=2) per step on "
              "oracle/_ref (unmodified reference sources, OpenBLAS 0.3.15); warm-up steps use an "
              "m=16 r=4 column")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded N(0,1) Box-Muller over SplitMix64)",
            "config": workload_config({"sample": "interior-column einsumsvd"}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if len(times) < args.steps:
        line["steps_note"] = f"timed {len(times)} of {args.steps} requested steps within the {budget:.0f} s budget"
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

    if dist:
        t = torch.tensor([dt, dt_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt, dt_e2e = float(t[0]), float(t[1])

    if rank != 0:
        return 0
    flops = alg_flops_row()
    value = world * flops / dt / 1e12
    peak = _fp64_peak()
    g = rep["gemm"]
    # achieved = real flops the DMMAs execute (3M launches: 6 per complex MAC,
    # 4M launches: 8) / device time -- the tensor-pipe roofline; the algorithmic
    # rate (8 per complex MAC, the reference's count) is reported beside it.
    achieved = g["exec_flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else None
    achieved_alg = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else None
    total_ms = sum(v["ms"] for v in rep.values())
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak["tflops"], "unit": "TFLOP/s",
            "frac": achieved / peak["tflops"] if achieved else None, "traffic": _ncu_traffic(),
            "kernel": "zgemm_cx_kernel (complex FP64 GEMM on DMMA.8x8x4: 3M/Gauss and 4M complex-fragment "
                      "instantiations, all launches of the step)",
            "achieved_algorithmic": achieved_alg,
            "kernel_share_of_step": g["ms"] / total_ms if total_ms else None,
            "profile_pass": "serialised (overlap off); the timed step overlaps the k x k eigensolver with GEMMs",
            "launches_per_step": g["launches"], "avg_launch_ms": g["ms"] / max(1, g["launches"]),
            "algorithmic_flops_per_step": g["flops"], "executed_flops_per_step": g["exec_flops"],
            "peak_source": peak["source"],
            "whole_step_frac": (flops / dt / 1e12) / peak["tflops"],
            "breakdown_ms": {k: round(v["ms"], 3) for k, v in rep.items()}}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded N(0,1) Box-Muller over SplitMix64)",
            "config": workload_config({"parallelism": f"replicas x{world}", "s_per_row_absorb": dt}),
            "clocks": clk.summary(), "gpu_launches": launches,
            "e2e": {"value": world * flops / dt_e2e / 1e12, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "s_per_step": dt_e2e},
            "roofline": roof}
    if world == 1 and not args.no_norms:
        line["s_per_norm"] = norm_timings(A, ctx)
    if world == 1 and not args.no_cpu_baseline:
        try:
            cores = os.cpu_count() or 1
            cdt, cfl = cpu_sample(cores)
            line["cpu_baseline"] = {"value": cfl / cdt / 1e12, "unit": UNIT, "cores": cores, "kind": "reference",
                                    "sample": "one interior-column einsumsvd of config 2 on oracle/_ref "
                                              f"({cdt:.1f} s)"}
        except Exception as e:  # oracle missing on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    return 0


def norm_timings(A, ctx):
    """The metric's other half: seconds per <psi|psi> by two-layer boundary
    contraction (contract_two_layer) on BASELINE configs 1, 3 and 5, and
    seconds per ITE step of config 4, through the public API (wall clock around
    synchronised calls; inputs resident).  Reference CPU figures for 3 and 5 are
    SURVEY §6's (1511 s for config 3's cache + bands on 8 cores; ~16 h per
    config-5 sweep); config 1's and 4's are timed by tools/bench_configs.py."""
    out = {}
    c1 = inputs.config1()
    st = A.PepsState(4, 4, 2, c1["sites"], ctx=ctx)
    o1 = A.ContractOption.two_layer_opt(4, c1["seed"], 1, 4)
    A.contract_two_layer(st, st, o1)
    t0 = time.perf_counter()
    for _ in range(10):
        A.contract_two_layer(st, st, o1)
    out["config1_4x4_r2_m4"] = (time.perf_counter() - t0) / 10
    for name, cfg, r, m, q, os_ in (("config3_16x16_r6_m36", inputs.config3(), 6, 36, 2, -1),
                                    ("config5_32x32_r8_m64", inputs.config5(), 8, 64, 2, 8)):
        n = cfg["rows"]
        st = A.PepsState(n, n, 2, cfg["sites"], ctx=ctx)
        opt = A.ContractOption.two_layer_opt(m, cfg["seed"], q, os_)
        reps = 3 if n <= 16 else 1  # config 3: warm-up + median of 3 (0.4 s each); config 5: one cold-ish shot
        if reps > 1:
            A.contract_two_layer(st, st, opt)
        ts = []
        for _ in range(reps):
            ctx.sync()
            t0 = time.perf_counter()
            A.contract_two_layer(st, st, opt)
            ts.append(time.perf_counter() - t0)
        out[name] = sorted(ts)[len(ts) // 2]
        del st
    plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
    st = A.PepsState(8, 8, 2, plus, ctx=ctx)
    A.ite_tfim(st, 1.0, 3.0, 0.01, 2, 8)
    ctx.sync()
    t0 = time.perf_counter()
    A.ite_tfim(st, 1.0, 3.0, 0.01, 20, 8)
    ctx.sync()
    out["config4_ite_8x8_r8_s_per_step"] = (time.perf_counter() - t0) / 20
    out["note"] = "seconds per norm (config 4: per Trotter step); wall clock, synchronised, one B200"
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
    """--sharded: ONE config-2 row absorb split across the N ranks along the
    boundary bond (paper_2006_15234_b200/sharded.py, NCCL collectives);
    scaling "strong", value = the row's algorithmic flops / max-over-ranks time."""
    import torch
    import torch.distributed as dist
    import paper_2006_15234_b200.api as A
    from paper_2006_15234_b200 import sharded as SH

    torch.cuda.set_device(local_rank)
    ctx = A.Context(local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local_rank))
    ops = SH.DeviceOps(SH.Comm(), ctx)
    c2 = inputs.config2(seed=2)
    row = [A.to_device(c2["sites"][1 * L + c], ctx) for c in range(L)]
    tops = [A.to_device(t, ctx) for t in c2["top"]]
    opt = A.ContractOption.two_layer_opt(M, c2["seed"], Q, OS)

    def step(tp, rw):
        return SH.sharded_two_layer_apply_row(ops, tp, c2["phys"], rw, rw, 1, M, opt.seed, Q, OS, True, 0x20)

    for _ in range(max(args.warmup, 0)):
        out = step(tops, row)
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
            out = step(tops, row)
        e1.record(stream)
        ctx.sync()
        torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / args.steps
    launches = ctx.counters()["launches"]
    # e2e: inputs from pinned host memory, boundary copied back every step
    pinned_in = [torch.from_numpy(np.ascontiguousarray(x).view(np.float64)).pin_memory()
                 for x in [c2["sites"][1 * L + c] for c in range(L)] + list(c2["top"])]
    shapes = [c2["sites"][1 * L + c].shape for c in range(L)] + [t.shape for t in c2["top"]]
    h2d = sum(p.numel() * 8 for p in pinned_in)
    d2h = 0
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        dev = [A.DeviceTensor(_from_pinned(ctx, p, sh), ctx) for p, sh in zip(pinned_in, shapes)]
        o, _ = step(dev[L:], dev[:L])
        host = [x.numpy() for x in o]
        d2h = sum(h.nbytes for h in host)
    ctx.sync()
    dt_e2e = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([dt, dt_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt, dt_e2e = float(t[0]), float(t[1])
    if rank != 0:
        return 0
    flops = alg_flops_row()
    line = {"metric": METRIC, "value": flops / dt / 1e12, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded N(0,1) Box-Muller over SplitMix64)",
            "config": workload_config({"parallelism": f"bond-sharded x{world} (t / s of the boundary bond)",
                                       "s_per_row_absorb": dt}),
            "clocks": clk.summary(), "gpu_launches": launches,
            "e2e": {"value": flops / dt_e2e / 1e12, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "s_per_step": dt_e2e}}
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
                    help="N>1: split one row absorb across the ranks along the boundary bond (strong scaling) "
                         "instead of N independent replicas")
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
        if args.sharded:
            return run_sharded(args, rank, world, local_rank)
        return run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
