"""Row-pipeline depth sweep (option pipeline_rows) for the config-3 and config-5 norms."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200 import inputs
ctx = A.default_context()
res = {}
for name, cfg, m, q, os_, depths in (("config3", inputs.config3(), 36, 2, -1, [2, 3, 4, 6, 8]),
                                     ("config5", inputs.config5(), 64, 2, 8, [2, 3, 4, 5])):
    n = cfg["rows"]
    st = A.PepsState(n, n, 2, cfg["sites"], ctx=ctx)
    opt = A.ContractOption.two_layer_opt(m, cfg["seed"], q, os_)
    for K in depths:
        ctx.set_option("pipeline_rows", K)
        v = A.contract_two_layer(st, st, opt)
        ctx.sync()
        ts = []
        for _ in range(2 if name == "config3" else 1):
            t0 = time.perf_counter()
            v2 = A.contract_two_layer(st, st, opt)
            ctx.sync()
            ts.append(time.perf_counter() - t0)
        res[f"{name}_K{K}"] = [min(ts), v2 == v]
    ctx.set_option("pipeline_rows", -1)
print(json.dumps(res))
