"""One config-2 row absorb (after one warm-up absorb) for ncu launch lists.

    python tools/prof_step.py            # plain run (must exit 0 before ncu)
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/prof_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2006_15234_b200.api as A  # noqa: E402
from paper_2006_15234_b200 import inputs  # noqa: E402

c2 = inputs.config2()
st = A.PepsState(3, 8, 2, c2["sites"])
top = A.TwoLayerBoundary.from_sites(c2["top"], c2["phys"])
opt = A.ContractOption.two_layer_opt(64, c2["seed"], 2, 8)
n = int(os.environ.get("PEPSB_PROF_STEPS", "2"))
ctx = A.default_context()
for i in range(n):
    ctx.reset_counters()
    out = A.two_layer_apply_row(top, st, st, 1, opt, 0x20)
    ctx.sync()
    print("step", i, ctx.counters(), flush=True)
