"""Developer tool: per-shape GEMM time in one config-2 row absorb (event-timed).

Runs one absorb with PEPSB_TRACE_GEMM (shapes to stderr) and the library's
per-launch event profile, then joins them in launch order."""
import os, re, subprocess, sys, json
if os.environ.get("_GS_CHILD") != "1":
    env = dict(os.environ, PEPSB_TRACE_GEMM="1", _GS_CHILD="1")
    r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
    shapes = [l for l in r.stderr.splitlines() if l.startswith("[zgemm]")]
    times = json.loads(r.stdout.strip().splitlines()[-1])
    n = len(times)
    shapes = shapes[-n:]
    agg = {}
    for s, t in zip(shapes, times):
        key = s[8:]
        a = agg.setdefault(key, [0, 0.0, 0.0])
        a[0] += 1; a[1] += t[0]; a[2] += t[1]
    tot = sum(v[1] for v in agg.values())
    print(f"GEMM total {tot:.2f} ms")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"{v[1]:8.2f} ms {v[0]:3d}x {v[2] / v[1] / 1e9:6.1f} TF  {k}")
    sys.exit(0)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200 import inputs
c2 = inputs.config2()
ctx = A.default_context()
st = A.PepsState(3, 8, 2, c2["sites"])
top = A.TwoLayerBoundary.from_sites(c2["top"], c2["phys"])
opt = A.ContractOption.two_layer_opt(64, c2["seed"], 2, 8)
A.two_layer_apply_row(top, st, st, 1, opt, 0x20); ctx.sync()
# per-launch list via a small extension of the profile: re-run with profiling, read per-record times
from paper_2006_15234_b200._lib import lib
ctx.profile(True)
A.two_layer_apply_row(top, st, st, 1, opt, 0x20)
recs = (C.c_double * (3 * 4096))()
n = lib().pepsb_ctx_profile_records(ctx.h, recs, 4096)
ctx.profile(False)
print(json.dumps([[recs[3 * i + 1], recs[3 * i + 2]] for i in range(n) if int(recs[3 * i]) == 0]))
