"""Config-4 ITE step time (device, warm) -- run under different env settings."""
import sys, time, numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2006_15234_b200.api as A
ctx = A.default_context()
plus = [np.array([1, 1], dtype=complex).reshape(2, 1, 1, 1, 1) / np.sqrt(2) for _ in range(64)]
s = A.ite_tfim(A.PepsState(8, 8, 2, plus), 1.0, 3.0, 0.01, 5, 8)
ctx.sync()
t0 = time.perf_counter()
out = A.ite_tfim(A.PepsState(8, 8, 2, plus), 1.0, 3.0, 0.01, 100, 8)
ctx.sync()
dt = (time.perf_counter() - t0) / 100
sites = [x.numpy() for x in out.sites]
print({"s_per_step": dt, "checksum": float(sum(np.abs(x).sum() for x in sites))})
