"""Developer tool: a few eigh cases (run under compute-sanitizer)."""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import paper_2006_15234_b200.api as A  # noqa: E402
from oracle import peps_oracle as O  # noqa: E402

ctx = A.default_context()
ctx.set_option("eig_solver", int(sys.argv[1]) if len(sys.argv) > 1 else 0)
for n in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["2", "5", "33", "72"])]:
    a = O.random_tensor((n, n), n)
    m = 0.5 * (a + a.conj().T)
    w, v = A.eigh(m)
    x = v.numpy()
    print(n, "val err %.2e" % np.abs(w - np.linalg.eigvalsh(m)[::-1]).max(),
          "res %.2e" % np.abs(m @ x - x * w).max(), "orth %.2e" % np.abs(x.conj().T @ x - np.eye(n)).max(), flush=True)
from paper_2006_15234_b200._lib import lib  # noqa: E402
for n in (16, 32, 64, 72, 128):
    a = O.random_tensor((n, n), n)
    m = 0.5 * (a + a.conj().T)
    for w in range(8, 40):
        lib().pepsb_ctx_debug_word(ctx.h, w, 1)
    ctx.profile(True)
    A.eigh(m)
    rep = ctx.profile_report()
    ctx.profile(False)
    words = [lib().pepsb_ctx_debug_word(ctx.h, w, 1) for w in range(8, 40)]
    print(n, "ms %.3f" % rep["small"]["ms"], "tri/dc/back kcyc", words[0:3], "block merge hcyc", words[4:8],
          "secular its/roots", words[16:18], flush=True)
