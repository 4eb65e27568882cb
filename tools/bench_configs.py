"""Per-config measurements of the einsumsvd path on one B200 (BASELINE configs 1, 3, 4, 5).

bench.py's headline line is config 2 (the metric's TF/s quote).  This tool times
the other BASELINE configs through the same public API and prints one JSON line
per config; results are committed under profiles/ (rNN_configs.jsonl).

  python tools/bench_configs.py [--configs 1,3,4,5] [--ref] [--zz all|centre]

--ref also runs the compiled reference (oracle/_ref, all host threads) where it
finishes in bounded time (config 1 norm; config 4 100-step ITE, compared
elementwise), as the parity/CPU-baseline leg.  Configs 3 and 5 are far beyond a
bounded CPU run (1511 s / ~16 h); their CPU numbers are the ones
measured in SURVEY §6 / BASELINE.md, and their parity is pinned by the reduced
size tests in tests/test_gpu_peps.py.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import paper_2006_15234_b200.api as A  # noqa: E402
from paper_2006_15234_b200 import costmodel, inputs  # noqa: E402

Z = np.diag([1.0, -1.0]).astype(complex)


def _sync(ctx):
    ctx.sync()


def zz_pieces():
    """split_two_site of Z (x) Z (observables.cpp:284-295) via the device SVD."""
    zz = np.einsum("ac,bd->abcd", Z, Z)
    u, s, v = A.svd(zz.transpose(0, 2, 1, 3).copy(), 2)
    s = np.asarray(s)
    g = int((s >= 1e-14 * s[0]).sum())
    w = np.sqrt(s[:g])
    left = u.numpy()[..., :g] * w
    right = (v.numpy()[:g] * w[:, None, None]).transpose(1, 2, 0)
    return left, right


def contract_flops(n, r, m, q, os_):
    """Algorithmic real FP64 flops (4 x the reference's instr::flops) of contract_two_layer's
    row absorbs on an n x n lattice whose boundary bonds are already m (true for configs 3
    and 5: the first row's boundary bond r*r equals m)."""
    return sum(4 * costmodel.two_layer_row_flops(n, r, m, q, os_, interior=row < n - 1) for row in range(1, n))


def bond_spectra(sites, rows, cols, top=8):
    """Gauge-invariant per-bond check: singular values of the two-site tensor
    contracted over each bond and matricised (site-a legs) x (site-b legs) --
    invariant under unitary gauge changes on every bond (the SVD phase and
    degenerate-subspace freedom of simple update), normalised by the largest."""
    out = []
    for r in range(rows):
        for c in range(cols):
            a = sites[r * cols + c]
            if c + 1 < cols:  # horizontal: a right (4) with b left (2)
                b = sites[r * cols + c + 1]
                m = np.tensordot(a, b, axes=([4], [2]))  # (pa, ua, la, da, pb, ub, db, rb)
                m = m.reshape(int(np.prod(a.shape[:4])), -1)
                s = np.linalg.svd(m, compute_uv=False)[:top]
                out.append(s / s[0])
            if r + 1 < rows:  # vertical: a down (3) with b up (1)
                b = sites[(r + 1) * cols + c]
                m = np.tensordot(a, b, axes=([3], [1]))
                m = m.reshape(int(np.prod(a.shape[:3]) * a.shape[4]), -1)
                s = np.linalg.svd(m, compute_uv=False)[:top]
                out.append(s / s[0])
    return out


def spectra_err(got, want, rows, cols):
    sg, sw = bond_spectra(got, rows, cols), bond_spectra(want, rows, cols)
    return max(float(np.abs(x - y).max()) for x, y in zip(sg, sw))


def cfg1(args, ctx):
    c = inputs.config1()
    st = A.PepsState(4, 4, 2, c["sites"], ctx=ctx)
    opt = A.ContractOption.two_layer_opt(4, c["seed"], 1, 4)
    for _ in range(3):
        v = A.contract_two_layer(st, st, opt)
    n = 20
    t0 = time.perf_counter()
    for _ in range(n):
        v = A.contract_two_layer(st, st, opt)
    dt = (time.perf_counter() - t0) / n
    exact = None
    out = {"config": 1, "workload": "4x4 r=2 PEPS norm, two-layer IBMPS m=4 os=4 q=1", "s_per_norm": dt,
           "norm": [v.real, v.imag]}
    if args.ref:
        from oracle import ref
        ref.set_threads(os.cpu_count() or 1)
        t0 = time.perf_counter()
        for _ in range(n):
            w, _ = ref.contract_two_layer(c["sites"], 4, 4, 4, c["seed"], 1, 4)
        out["ref_s_per_norm"] = (time.perf_counter() - t0) / n
        out["ref_norm"] = [w.real, w.imag]
        out["rel_err_vs_ref"] = abs(v - w) / abs(w)
        exact = ref.inner_exact(c["sites"], 4, 4)
        out["exact"] = [exact.real, exact.imag]
        out["truncation_rel_diff_vs_exact"] = abs(v - exact) / abs(exact)
        out["cpu_cores"] = os.cpu_count()
    return out


def cfg3(args, ctx):
    c = inputs.config3()
    n = c["rows"]
    st = A.PepsState(n, n, 2, c["sites"], ctx=ctx)
    opt = A.ContractOption.two_layer_opt(c["m"], c["seed"], c["power_iters"], c["oversample"])
    A.contract_two_layer(st, st, opt)  # warm-up (pools, helper contexts, plans)
    A.build_row_cache(st, opt)
    _sync(ctx)
    t_norm, t_cache = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        nrm = A.contract_two_layer(st, st, opt)
        t_norm.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        cache = A.build_row_cache(st, opt)
        _sync(ctx)
        t_cache.append(time.perf_counter() - t0)
    t_norm, t_cache = sorted(t_norm)[1], sorted(t_cache)[1]  # medians of 3 warm runs
    norm = A.chain_scalar(cache.tops[n - 1])
    t0 = time.perf_counter()
    zs = np.zeros((n, n))
    for i in range(n):
        top = cache.tops[i - 1] if i > 0 else None
        bot = cache.bots[i + 1] if i + 1 < n else None
        env = A.band_environment(top, st, st, i, i, bot)
        for j in range(n):
            val = A.band_splice(env, top, st, st, bot, [A.InsertionPiece((i, j), Z, [])], j, j) / norm
            zs[i, j] = val.real
    t_bands = time.perf_counter() - t0
    return {"config": 3, "norm_alg_tflops": contract_flops(n, 6, 36, 2, 5) / t_norm / 1e12, "workload": "16x16 r=6 m=36 (k=41, q=2): norm + <Z_i> on all 256 sites via cached envs",
            "s_per_norm": t_norm, "norm": [nrm.real, nrm.imag], "cache_s": t_cache,
            "bands_256_Z_s": t_bands, "total_cached_s": t_cache + t_bands,
            "cached_norm_bitwise_equal": bool(norm == nrm), "mean_Z": float(zs.mean()),
            "Z_centre": float(zs[n // 2, n // 2]),
            "ref_cpu_s_total_SURVEY": 1511.1, "ref_cpu_cores_SURVEY": 8}


def cfg4(args, ctx):
    steps = args.ite_steps
    plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
    st = A.PepsState(8, 8, 2, plus, ctx=ctx)
    A.ite_tfim(st, 1.0, 3.0, 0.01, 2, 8)  # warm-up
    _sync(ctx)
    ctx.reset_counters()
    t0 = time.perf_counter()
    out = A.ite_tfim(st, 1.0, 3.0, 0.01, steps, 8)
    _sync(ctx)
    dt = time.perf_counter() - t0
    degenerate = ctx.counter("degenerate_truncations")
    res = {"config": 4, "workload": f"TFIM ITE 8x8 r=8 J=1 h=3 tau=0.01, {steps} steps, simple update "
                                     "(bonds batched per colour)",
           "s_total": dt, "s_per_step": dt / steps, "updates_per_s": steps * (64 + 112) / dt,
           "degenerate_truncations": degenerate, "bond_updates": steps * 112}
    if args.ref:
        from oracle import ref
        ref.set_threads(os.cpu_count() or 1)
        t0 = time.perf_counter()
        want, _ = ref.ite_tfim(plus, 8, 8, 1.0, 3.0, 0.01, steps, 8)
        rdt = time.perf_counter() - t0
        got = [s.numpy() for s in out.sites]
        shapes_equal = [g.shape for g in got] == [w.shape for w in want]
        worst = max(float(np.abs(g - w).max() / max(np.abs(w).max(), 1e-300)) for g, w in zip(got, want)) \
            if shapes_equal else None
        rs = np.random.default_rng(45)
        pert = [x * (1.0 + 1e-14 * rs.standard_normal()) for x in plus]
        want2, _ = ref.ite_tfim(pert, 8, 8, 1.0, 3.0, 0.01, steps, 8)
        if [w.shape for w in want2] == [w.shape for w in want]:
            res["ref_vs_ref_perturbed_1e-14_bond_spectra_err"] = spectra_err(want2, want, 8, 8)
        res.update({"ref_s_total": rdt, "ref_s_per_step": rdt / steps, "cpu_cores": os.cpu_count(),
                    "shapes_bit_exact": shapes_equal, "max_site_rel_err_vs_ref": worst,
                    "bond_spectra_max_err_vs_ref": spectra_err(got, want, 8, 8) if shapes_equal else None})
        # Gauge-invariant comparison: the SVD gauge of degenerate bond spectra
        # (exact at the |+> start) is arbitrary, so compare the STATES: norms and
        # fidelity |<ref|gpu>|^2 / (<ref|ref><gpu|gpu>) by device boundary
        # contraction (m=64, accurate for this weakly entangled state).
        # The unnormalised states reach |<psi|psi>| ~ 1e300+ after 100 steps (the
        # reference does not normalise either): scale every site by its max |entry|
        # and carry the log of the scale factors.
        mg = [float(np.abs(g).max()) for g in got]
        mr = [float(np.abs(w).max()) for w in want]
        sg = A.PepsState(8, 8, 2, [g / m for g, m in zip(got, mg)], ctx=ctx)
        sr = A.PepsState(8, 8, 2, [w / m for w, m in zip(want, mr)], ctx=ctx)
        opt = A.ContractOption.two_layer_opt(64, 7, 2, 8)
        n_g = A.contract_two_layer(sg, sg, opt)
        n_r = A.contract_two_layer(sr, sr, opt)
        ov = A.contract_two_layer(sr, sg, opt)
        ln_g = np.log(abs(n_g)) + 2 * np.log(mg).sum()
        ln_r = np.log(abs(n_r)) + 2 * np.log(mr).sum()
        res.update({"log_norm_gpu_state": ln_g, "log_norm_ref_state": ln_r,
                    "log_norm_rel_diff": abs(ln_g - ln_r) / abs(ln_r),
                    "norm_rel_diff": float(abs(np.expm1(ln_g - ln_r))),
                    "one_minus_fidelity": 1.0 - abs(ov) ** 2 / (abs(n_g) * abs(n_r))})
    return res


def cfg4b(args, ctx):
    """Config 4 from a random (symmetry-breaking) product state: the |+> start of
    config 4 produces exactly degenerate bond spectra whose truncation subspace
    is rounding-dependent, so bond-for-bond parity is checked here,
    elementwise, on the full 8x8 r=8 100-step evolution."""
    steps = args.ite_steps
    rs = np.random.default_rng(44)
    init = []
    for _ in range(64):
        v = rs.standard_normal(2) + 1j * rs.standard_normal(2)
        init.append((v / np.linalg.norm(v)).reshape(2, 1, 1, 1, 1))
    st = A.PepsState(8, 8, 2, init, ctx=ctx)
    _sync(ctx)
    t0 = time.perf_counter()
    ctx.reset_counters()
    out = A.ite_tfim(st, 1.0, 3.0, 0.01, steps, 8)
    _sync(ctx)
    dt = time.perf_counter() - t0
    res = {"config": "4b", "degenerate_truncations": ctx.counter("degenerate_truncations"), "workload": f"as config 4 from a random product state, {steps} steps", "s_total": dt,
           "s_per_step": dt / steps}
    from oracle import ref
    ref.set_threads(os.cpu_count() or 1)
    want, _ = ref.ite_tfim(init, 8, 8, 1.0, 3.0, 0.01, steps, 8)
    got = [s.numpy() for s in out.sites]
    shapes_equal = [g.shape for g in got] == [w.shape for w in want]
    res["shapes_bit_exact"] = shapes_equal
    if shapes_equal:
        res["max_site_rel_err_vs_ref"] = max(float(np.abs(g - w).max() / np.abs(w).max()) for g, w in zip(got, want))
        res["bond_spectra_max_err_vs_ref"] = spectra_err(got, want, 8, 8)
    # intrinsic sensitivity: the reference against itself with the initial state
    # perturbed at 1e-14 relative (the spread any two correct implementations
    # with different rounding can show after 100 steps)
    pert = [x * (1.0 + 1e-14 * rs.standard_normal()) for x in init]
    want2, _ = ref.ite_tfim(pert, 8, 8, 1.0, 3.0, 0.01, steps, 8)
    if [w.shape for w in want2] == [w.shape for w in want]:
        res["ref_vs_ref_perturbed_1e-14_bond_spectra_err"] = spectra_err(want2, want, 8, 8)
    return res


def cfg5(args, ctx):
    c = inputs.config5()
    n = c["rows"]
    st = A.PepsState(n, n, 2, c["sites"], ctx=ctx)
    opt = A.ContractOption.two_layer_opt(c["m"], c["seed"], c["power_iters"], c["oversample"])
    t0 = time.perf_counter()
    nrm = A.contract_two_layer(st, st, opt)
    t_norm = time.perf_counter() - t0
    res = {"config": 5, "workload": "32x32 r=8 m=64 (k=72, q=2): norm by two-layer boundary contraction "
                                    "+ nearest-neighbour ZZ via cached envs",
           "s_per_norm": t_norm, "norm": [nrm.real, nrm.imag],
           "norm_alg_flops_model": contract_flops(n, 8, 64, 2, 8),
           "norm_alg_tflops": contract_flops(n, 8, 64, 2, 8) / t_norm / 1e12}
    if args.zz == "none":
        return res
    t0 = time.perf_counter()
    cache = A.build_row_cache(st, opt)
    _sync(ctx)
    res["cache_s"] = time.perf_counter() - t0
    norm = A.chain_scalar(cache.tops[n - 1])
    res["cached_norm_bitwise_equal"] = bool(norm == nrm)
    left, right = zz_pieces()
    i, j = n // 2, n // 2 - 1
    t0 = time.perf_counter()
    top, bot = cache.tops[i - 1], cache.bots[i + 1]
    env = A.band_environment(top, st, st, i, i, bot)
    pieces = [A.InsertionPiece((i, j), left, [0]), A.InsertionPiece((i, j + 1), right, [0])]
    zz_h = A.band_splice(env, top, st, st, bot, pieces, j, j + 1) / norm
    res["zz_centre_horizontal"] = [zz_h.real, zz_h.imag]
    res["zz_centre_horizontal_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    top, bot = cache.tops[i - 1], cache.bots[i + 2]
    env2 = A.band_environment(top, st, st, i, i + 1, bot)
    pieces = [A.InsertionPiece((i, j), left, [0]), A.InsertionPiece((i + 1, j), right, [0])]
    zz_v = A.band_splice(env2, top, st, st, bot, pieces, j, j) / norm
    res["zz_centre_vertical"] = [zz_v.real, zz_v.imag]
    res["zz_centre_vertical_s"] = time.perf_counter() - t0
    return res


def cfg_sens(args, ctx):
    """Rounding sensitivity of truncated boundary contractions.  Reduced size
    (8x8 r=4 m=16 q=2 os=4, within the reference's reach): device vs
    reference, and reference vs itself after a 1e-14 relative perturbation of
    every site; full config 5: device with two rounding-different schedules
    (eigensolver/apply overlap on vs off)."""
    from oracle import ref
    ref.set_threads(os.cpu_count() or 1)
    out = {"config": "sensitivity"}
    sites = inputs.random_peps(8, 8, 4, 51, scale=1 / np.sqrt(32))
    st = A.PepsState(8, 8, 2, sites, ctx=ctx)
    opt = A.ContractOption.two_layer_opt(16, 9, 2, 4)
    dev = A.contract_two_layer(st, st, opt)
    w, _ = ref.contract_two_layer(sites, 8, 8, 16, 9, 2, 4)
    rs = np.random.default_rng(3)
    pert = [x * (1.0 + 1e-14 * rs.standard_normal()) for x in sites]
    w2, _ = ref.contract_two_layer(pert, 8, 8, 16, 9, 2, 4)
    out.update({"reduced_8x8_r4_m16_device_vs_ref": abs(dev - w) / abs(w),
                "reduced_8x8_r4_m16_ref_vs_ref_perturbed_1e-14": abs(w2 - w) / abs(w)})
    c = inputs.config5()
    st = A.PepsState(32, 32, 2, c["sites"], ctx=ctx)
    opt = A.ContractOption.two_layer_opt(64, c["seed"], 2, 8)
    a = A.contract_two_layer(st, st, opt)
    ctx.set_option("overlap", 0)
    b = A.contract_two_layer(st, st, opt)
    ctx.set_option("overlap", 1)
    out["config5_overlap_on_vs_off"] = abs(a - b) / abs(b)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--ite-steps", type=int, default=100)
    ap.add_argument("--zz", choices=["none", "centre"], default="centre")
    args = ap.parse_args()
    ctx = A.default_context()
    fns = {"1": cfg1, "3": cfg3, "4": cfg4, "4b": cfg4b, "5": cfg5, "sens": cfg_sens}
    for k in args.configs.split(","):
        t0 = time.perf_counter()
        res = fns[k](args, ctx)
        res["wall_s"] = time.perf_counter() - t0
        res["launches"] = ctx.counters().get("launches")
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
