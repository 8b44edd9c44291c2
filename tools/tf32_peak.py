"""Measured TF32 tensor peak of this B200 (the roofline denominator for the NCC Gram).

MEASURED_PEAKS.json (driver-written) carries HBM and dense BF16 only.  This
measures, the same way the driver does for BF16 (torch.matmul at 8192^3,
2*N^3 flops, CUDA events): TF32 (fp32 inputs with allow_tf32, cuBLAS picks a
tcgen05 kind::tf32 kernel) burst = best of 10 and sustained = back to back for
4 s, plus BF16 as a same-box cross-check against MEASURED_PEAKS.json.

  python tools/tf32_peak.py > profiles/r2_tf32_peak.json
"""

from __future__ import annotations

import json
import subprocess
import time

import torch


def measure(dtype, n=8192, reps=10, sustain_s=4.0):
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flops = 2.0 * n ** 3
    cnt = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    while time.perf_counter() - t0 < sustain_s:
        for _ in range(10):
            a @ b
        cnt += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = flops * cnt / (e0.elapsed_time(e1) / 1e3) / 1e12
    return {"burst_tflops": flops / (best / 1e3) / 1e12, "sustained_tflops": sus, "n": n}


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    out = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": "torch.matmul 8192^3 (2*N^3 flops), CUDA events; burst = best of 10, sustained = 4 s back to back",
           "tf32": measure(torch.float32), "bf16": measure(torch.bfloat16)}
    try:
        out["clocks"] = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw",
                                        "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    except Exception:
        pass
    print(json.dumps(out))


if __name__ == "__main__":
    main()
