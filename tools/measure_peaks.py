"""FP64 and TF32 dense matmul peaks on this B200, measured like
MEASURED_PEAKS.json's bf16 figure (torch.matmul 8192^3, best of 10 with CUDA
events; 2 N^3 flop), plus FP64 SIMT FMA throughput from a DFMA-chain kernel
(torch's fp64 GEMM may use DMMA).  SURVEY.md 8(d) asks for these before any
fp64 / tf32 kernel is quoted against a roofline."""
import json, os, sys
import torch


def mm_peak(dtype, tf32=False, N=8192, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(N, N, device="cuda", dtype=dtype)
    b = torch.randn(N, N, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2.0 * N ** 3 / (best / 1e3) / 1e12


out = {"fp64_matmul_tflops": mm_peak(torch.float64),
       "tf32_matmul_tflops": mm_peak(torch.float32, tf32=True),
       "fp32_simt_matmul_tflops": mm_peak(torch.float32, tf32=False),
       "how": "torch.matmul 8192^3 (2 N^3 flop), best of 10, CUDA events; tf32 via allow_tf32",
       "gpu": torch.cuda.get_device_name()}
print(json.dumps(out))
