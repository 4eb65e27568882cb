"""A/B of a context option on the s/norm of configs 1, 3, 5 (and one config-2 row):
  python tools/opt_ab.py <option> <a> <b>"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200 import inputs
name, va, vb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
ctx = A.default_context()
res = {"option": name, "values": [va, vb]}
c1 = inputs.config1()
cases = [("config1", A.PepsState(4, 4, 2, c1["sites"]), A.ContractOption.two_layer_opt(4, c1["seed"], 1, 4), 20)]
c3 = inputs.config3()
cases.append(("config3", A.PepsState(16, 16, 2, c3["sites"]), A.ContractOption.two_layer_opt(36, c3["seed"], 2, -1), 3))
c5 = inputs.config5()
cases.append(("config5", A.PepsState(32, 32, 2, c5["sites"]), A.ContractOption.two_layer_opt(64, c5["seed"], 2, 8), 1))
for cname, st, opt, reps in cases:
    out = []
    for v in (va, vb):
        ctx.set_option(name, v)
        A.contract_two_layer(st, st, opt)
        ctx.sync()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            A.contract_two_layer(st, st, opt)
            ctx.sync()
            ts.append(time.perf_counter() - t0)
        out.append(sorted(ts)[len(ts) // 2])
    res[cname] = out
print(json.dumps(res))
