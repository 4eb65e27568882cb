"""Measures the B200 FP64 roofline denominators (MEASURED_PEAKS.json has none).

- DMMA / DFMA issue ceilings from tools/fp64_probe.so (register-resident loops);
- cuBLAS DGEMM and ZGEMM throughput (torch.matmul float64 / complex128, 8192^3,
  best of 5, CUDA events) — the library-GEMM reference point.
Writes profiles/fp64_peak.json.
"""
import ctypes, json, os, sys, time
import torch

here = os.path.dirname(os.path.abspath(__file__))
res = (ctypes.c_double * 2)(0.0, 0.0)
lib = ctypes.CDLL(os.path.join(here, "fp64_probe.so"))
rc = lib.probe(res)
out = {"dmma_issue_tflops": res[0], "dfma_issue_tflops": res[1], "probe_rc": rc}
r16 = (ctypes.c_double * 3)(0.0, 0.0, 0.0)
out["probe16_rc"] = lib.probe16(r16)
out["dmma_m16n8k4_tflops"], out["dmma_m16n8k8_tflops"], out["dmma_m16n8k16_tflops"] = r16[0], r16[1], r16[2]

def gemm_tf(dtype, n, flop_per_mac):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return flop_per_mac * n ** 3 / best / 1e12

out["cublas_dgemm_tflops"] = gemm_tf(torch.float64, 8192, 2)
out["cublas_zgemm_tflops"] = gemm_tf(torch.complex128, 8192, 8)
out["gpu"] = torch.cuda.get_device_name(0)
out["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
print(json.dumps(out))
os.makedirs(os.path.join(here, "..", "gpurun_out"), exist_ok=True)
with open(os.path.join(here, "..", "gpurun_out", "fp64_peak.json"), "w") as f:
    json.dump(out, f, indent=1)
