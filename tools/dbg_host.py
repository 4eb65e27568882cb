"""Developer tool: wall time vs summed kernel time of one config-2 row absorb."""
import sys, time; sys.path.insert(0,'.')
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200 import inputs
c2 = inputs.config2()
ctx = A.default_context()
st = A.PepsState(3, 8, 2, c2["sites"])
top = A.TwoLayerBoundary.from_sites(c2["top"], c2["phys"])
opt = A.ContractOption.two_layer_opt(64, c2["seed"], 2, 8)
out = A.two_layer_apply_row(top, st, st, 1, opt, 0x20); ctx.sync()
for i in range(3):
    t0 = time.perf_counter(); out = A.two_layer_apply_row(top, st, st, 1, opt, 0x20); ctx.sync(); t1 = time.perf_counter()
    print("wall ms", (t1 - t0) * 1e3, flush=True)
ctx.profile(True)
t0 = time.perf_counter(); out = A.two_layer_apply_row(top, st, st, 1, opt, 0x20); ctx.sync(); t1 = time.perf_counter()
rep = ctx.profile_report(); ctx.profile(False)
print("profiled wall ms", (t1 - t0) * 1e3, {k: round(v["ms"], 2) for k, v in rep.items()})
from paper_2006_15234_b200._lib import lib
lib().pepsb_ctx_debug_word(ctx.h, 7, 1)
out = A.two_layer_apply_row(top, st, st, 1, opt, 0x20); ctx.sync()
print("total Jacobi sweeps in one row absorb:", lib().pepsb_ctx_debug_word(ctx.h, 7, 1))
