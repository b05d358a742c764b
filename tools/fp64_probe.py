"""Measure the FP64 roofline denominator on the GPU box and write
profiles/fp64_peak.json: cuBLAS DGEMM (torch.matmul float64, the library
analogue of MEASURED_PEAKS.json's cuBLAS bf16 figure) plus the DFMA / DMMA
microbenchmarks of tools/fp64_peak.cu."""
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dgemm_tflops(n=8192, reps=10):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return 2 * n ** 3 / best / 1e12


def main():
    out = {}
    binp = os.path.join(ROOT, "tools", "fp64_peak")
    if not os.path.exists(binp):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", binp,
                        os.path.join(ROOT, "tools", "fp64_peak.cu")], check=True)
    res = subprocess.run([binp], capture_output=True, text=True, check=True)
    out.update(json.loads(res.stdout))
    out["dgemm_cublas_tflops"] = dgemm_tflops()
    out["dgemm_cublas_tflops_4096"] = dgemm_tflops(4096)
    out["how"] = ("torch.matmul float64 8192^3 best of 10 (cuBLAS DGEMM); tools/fp64_peak.cu: 148x8 CTAs "
                  "x 256 threads of independent DFMA chains / mma.sync m8n8k4 f64 accumulators, best of 5")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
