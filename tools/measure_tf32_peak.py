"""Measures the dense TF32 tensor-core peak of this B200 with cuBLAS
(torch.matmul on fp32 with TF32 enabled, 8192^3, 2*N^3 flop), the
denominator of the join screen's roofline (MEASURED_PEAKS.json only has
bf16).  Same method as the driver's bf16 figure: best of 10 (burst) and
back to back for ~4 s (sustained).  Writes profiles/peaks_tf32.json."""

import json
import os
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    burst = 2 * n ** 3 / (best * 1e-3) / 1e12
    t0 = time.time()
    k = 0
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < 4.0:
        a @ b
        k += 1
        if k % 20 == 0:
            torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    sustained = 2 * n ** 3 * k / (s.elapsed_time(e) * 1e-3) / 1e12
    # fp64 (CUDA-core / DMMA) for the exact re-check's context
    a64, b64 = a[:4096, :4096].double(), b[:4096, :4096].double()
    a64 @ b64
    torch.cuda.synchronize()
    s.record()
    a64 @ b64
    e.record()
    torch.cuda.synchronize()
    f64 = 2 * 4096 ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12
    out = {"tf32_tflops": burst, "tf32_tflops_sustained": sustained, "fp64_tflops": f64,
           "gpu": torch.cuda.get_device_name(), "how": "torch.matmul fp32 allow_tf32 8192^3 best of 10; "
           "sustained = back to back 4 s; fp64 4096^3 single run", "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "peaks_tf32.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
