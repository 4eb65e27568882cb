"""Where does a config-2 row absorb spend its time with the streams overlapped?

Profiles one row absorb with the eigensolver/apply overlap ON (per-launch CUDA
events on whichever stream a kernel is enqueued on; pepsb_ctx_profile_timeline)
and prints: wall span, busy time per stream, the union (any kernel running),
the idle gaps (no kernel on either stream), and how the main-stream (latency
chain) time splits by kind while the side stream is idle.  The events add a
little per-launch overhead; use the shares, not the absolute span.

  python tools/timeline.py [--config 2|3|5] [--json out.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2006_15234_b200.api as A  # noqa: E402
from paper_2006_15234_b200 import inputs  # noqa: E402


def union_len(iv):
    iv = sorted(iv)
    tot, cs, ce = 0.0, None, None
    for s, e in iv:
        if cs is None or s > ce:
            if cs is not None:
                tot += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if cs is not None:
        tot += ce - cs
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    ctx = A.default_context()
    if a.config == 2:
        c = inputs.config2()
        sites, top, phys, m, os_ = c["sites"], c["top"], c["phys"], 64, 8
        L = 8
    else:
        L, bond, m, os_ = (16, 6, 36, -1) if a.config == 3 else (32, 8, 64, 8)
        scale = 1.0 / np.sqrt(bond * bond * 2)
        sites = inputs.random_peps(3, L, bond, 11, scale=scale)
        top, phys = inputs.random_boundary(L, (bond, bond), m, inputs.derive_seed(11, 0x70), scale=0.1)
    st = A.PepsState(3, L, 2, sites)
    tb = A.TwoLayerBoundary.from_sites(top, phys)
    opt = A.ContractOption.two_layer_opt(m, 2, 2, os_)
    for _ in range(2):
        A.two_layer_apply_row(tb, st, st, 1, opt, 0x20)
    ctx.sync()
    ctx.profile(True)
    A.two_layer_apply_row(tb, st, st, 1, opt, 0x20)
    tl = ctx.profile_timeline()
    ctx.profile(False)
    span = max(e for _, _, e, _, _ in tl) - min(s for _, s, _, _, _ in tl)
    main = [(s, e) for k, s, e, f, sd in tl if sd == 0]
    side = [(s, e) for k, s, e, f, sd in tl if sd == 1]
    busy_main, busy_side = union_len(main), union_len(side)
    busy_any = union_len(main + side)
    # main-stream kernels while the side stream is idle: the exposed latency chain
    side_iv = sorted(side)

    def overlap_with_side(s, e):
        tot = 0.0
        for a0, a1 in side_iv:
            if a1 <= s or a0 >= e:
                continue
            tot += min(e, a1) - max(s, a0)
        return tot

    exposed = {}
    alone = {}
    for k, s, e, f, sd in tl:
        if sd == 0:
            x = (e - s) - overlap_with_side(s, e)
            exposed[k] = exposed.get(k, 0.0) + x
        alone[k] = alone.get(k, 0.0) + (e - s)
    out = {"config": a.config, "launches": len(tl), "span_ms": span, "busy_main_ms": busy_main,
           "busy_side_ms": busy_side, "busy_any_ms": busy_any, "idle_ms": span - busy_any,
           "main_exposed_ms_by_kind": exposed, "serial_ms_by_kind": alone}
    print(json.dumps(out, indent=1))
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"summary": out, "timeline": tl}, f)


if __name__ == "__main__":
    main()
