"""Measure the B200 FP64 roofline denominators: torch (cuBLAS) DGEMM 8192^3
best-of-10 and sustained, plus the DFMA and DMMA pipes (tools/fp64_peak.cu)."""
import ctypes, json, os, subprocess, sys, time
import torch

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "libfp64_peak.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(here, "fp64_peak.cu")])
lib = ctypes.CDLL(so)
res = (ctypes.c_double * 2)()
lib.fp64_peak(res)
N = 8192
a = torch.randn(N, N, dtype=torch.float64, device="cuda")
b = torch.randn(N, N, dtype=torch.float64, device="cuda")
for _ in range(2):
    a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
t0 = time.time(); k = 0
e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True); e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; k += 1
e1.record(); torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / k
out = {"dgemm_tflops_burst": 2 * N**3 / (best * 1e-3) / 1e12, "dgemm_tflops_sustained": 2 * N**3 / (sus * 1e-3) / 1e12,
       "dfma_tflops": res[0], "dmma_tflops": res[1]}
print(json.dumps(out))
