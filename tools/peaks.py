"""Measure the compute peaks bench.py divides by (BASELINE.md asks for measured TF32
and FP32 peaks, measured "the way MEASURED_PEAKS measured bf16"):

  * cuBLAS GEMMs through torch.matmul, 8192^3, best of 10 (burst) and back to back
    for ~4 s (sustained): TF32 (allow_tf32) and plain FP32 (CUDA-core SGEMM);
  * tools/peaks.cu: FFMA, DMMA and the tcgen05 kind::tf32 issue ceiling.

Writes profiles/measured_compute_peaks.json (and prints it).
"""
import json
import os
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gemm(tf32: bool, n=8192, sustain_s=4.0):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, t0 = 0, time.time()
    e0.record()
    while time.time() - t0 < sustain_s:
        for _ in range(10):
            c = a @ b
        reps += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    fl = 2.0 * n ** 3
    del c
    return fl / best / 1e9, fl * reps / e0.elapsed_time(e1) / 1e9


def main():
    out = {"how": "cuBLAS via torch.matmul 8192^3 (2 N^3 flop): best of 10 and ~4 s back to back; "
                  "tools/peaks.cu microkernels (FFMA chains, DMMA m8n8k4, tcgen05 kind::tf32 M128 N256 "
                  "from shared memory, one CTA per SM)",
           "gpu": torch.cuda.get_device_name(0), "torch": torch.__version__,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    out["cublas_tf32_tflops"], out["cublas_tf32_tflops_sustained"] = gemm(True)
    out["cublas_fp32_tflops"], out["cublas_fp32_tflops_sustained"] = gemm(False)
    exe = "/tmp/tk_peaks"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                    os.path.join(ROOT, "tools", "peaks.cu"), "-lcuda"], check=True)
    mk = json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)
    out.update(mk)
    path = os.path.join(ROOT, "profiles", "measured_compute_peaks.json")
    if len(sys.argv) > 1:
        path = sys.argv[1]
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
