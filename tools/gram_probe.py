"""Developer tool: three Gram launches G = Z^H Z (Z 262144 x 72) with the Hermitian Gram kernel, for
    ncu --set full --import-source on --clock-control none -k regex:gram_ -c 3 python tools/gram_probe.py"""
import sys; sys.path.insert(0, '.')
import paper_2006_15234_b200.api as A
ctx = A.default_context()
ctx.set_option("gemm_gram", 1)
z = A.random_tensor((262144, 72), 21)
for _ in range(3):
    g = A.gram(z)
ctx.sync()
