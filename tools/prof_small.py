"""Launch-list driver for the latency-bound configs: one config-1 norm and
two config-4 ITE steps (after warm-ups), for
  ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_small.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_15234_b200.api as A  # noqa: E402
from paper_2006_15234_b200 import inputs  # noqa: E402

ctx = A.default_context()
which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("1", "both"):
    c1 = inputs.config1()
    st = A.PepsState(4, 4, 2, c1["sites"])
    o1 = A.ContractOption.two_layer_opt(4, c1["seed"], 1, 4)
    A.contract_two_layer(st, st, o1)
    ctx.sync()
    ctx.reset_counters()
    t0 = time.perf_counter()
    A.contract_two_layer(st, st, o1)
    ctx.sync()
    print("config1", time.perf_counter() - t0, ctx.counters()["launches"], flush=True)
if which in ("4", "both"):
    plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
    s4 = A.ite_tfim(A.PepsState(8, 8, 2, plus), 1.0, 3.0, 0.01, 20, 8)
    ctx.sync()
    ctx.reset_counters()
    t0 = time.perf_counter()
    A.ite_tfim(s4, 1.0, 3.0, 0.01, 2, 8)
    ctx.sync()
    print("config4 2 steps", time.perf_counter() - t0, ctx.counters()["launches"], flush=True)
