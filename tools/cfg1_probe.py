"""Config 1: wall time vs device busy time per norm (host-bound?)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200 import inputs
ctx = A.default_context()
c1 = inputs.config1()
st = A.PepsState(4, 4, 2, c1["sites"])
o1 = A.ContractOption.two_layer_opt(4, c1["seed"], 1, 4)
for _ in range(3):
    A.contract_two_layer(st, st, o1)
ctx.sync()
t0 = time.perf_counter(); A.contract_two_layer(st, st, o1); ctx.sync(); wall = time.perf_counter() - t0
ctx.profile(True)
A.contract_two_layer(st, st, o1)
tl = ctx.profile_timeline()
ctx.profile(False)
busy = sum(e - s for k, s, e, f, sd in tl)
span = max(e for _, _, e, _, _ in tl) - min(s for _, s, _, _, _ in tl)
byk = {}
for k, s, e, f, sd in tl:
    byk[k] = byk.get(k, 0) + (e - s)
os.environ["PEPSB_TRACE"] = "1"
print(json.dumps({"wall_ms": wall * 1e3, "profiled_launches": len(tl), "device_busy_ms": busy, "span_ms": span,
                  "by_kind_ms": byk, "counters": ctx.counters()}))
