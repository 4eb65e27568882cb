"""Developer tool: k x k eigensolver phase cycles (status words 8..10: tridiagonalisation, divide and
conquer, back-transformation in kcycles; 12..20: phases of the top-level merge, 21..28: per tree depth, 29..35: tridiagonalisation sections,
both in units of 16 cycles) and time per call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2006_15234_b200.api as A
from paper_2006_15234_b200._lib import lib
from oracle import peps_oracle as O
ctx = A.default_context()
REP = 10
for n in (16, 32, 41, 64, 72):
    a = O.random_tensor((3 * n, n), n)
    g = a.conj().T @ a
    for _ in range(3):
        A.gram_factors(g)
    for w in range(8, 40):
        lib().pepsb_ctx_debug_word(ctx.h, w, 1)
    ctx.profile(True)
    for _ in range(REP):
        A.gram_factors(g)
    rep = ctx.profile_report()
    ctx.profile(False)
    ms = rep["small"]["ms"] / max(1, rep["small"]["launches"])
    st = [lib().pepsb_ctx_debug_word(ctx.h, w, 1) / REP for w in (8, 9, 10)]
    mg = [lib().pepsb_ctx_debug_word(ctx.h, w, 1) * 16 / 1000 / REP for w in range(12, 21)]
    dp = [lib().pepsb_ctx_debug_word(ctx.h, w, 1) * 16 / 1000 / REP for w in range(21, 29)]
    print(f"n={n} {ms:.4f} ms  kcycles: tridiag {st[0]:.0f} dc {st[1]:.0f} back {st[2]:.0f}", flush=True)
    print("   top merge kcycles [z/perm, gather, deflate, rot, secular, zh, vectors, gemm, copy]:", " ".join(f"{x:.1f}" for x in mg))
    tp = [lib().pepsb_ctx_debug_word(ctx.h, w, 1) * 16 / 1000 / REP for w in range(29, 36)]
    print("   tridiag kcycles [matvec-wait + h-reduce, w+sync, x+norm, scalars, vnew, barrier 1, (clock skew)]:", " ".join(f"{x:.1f}" for x in tp))
    it = [lib().pepsb_ctx_debug_word(ctx.h, w, 1) for w in (36, 37, 38)]
    print(f"   secular iterations: max {it[0]}, mean {it[1] / max(1, it[2]):.2f} over {it[2] // REP} roots per call")
    print("   per depth kcycles (0 = top):", " ".join(f"{x:.1f}" for x in dp), flush=True)
