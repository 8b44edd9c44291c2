"""NCC all-pairs through the tcgen05 Gram kernel: time, TF32 TFLOP/s, accuracy vs the fp32 per-pair path.

  python tools/ncc_bench.py [n] [side]
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2009_04755_b200 import _lib, device


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    side = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    d = side * side
    items = torch.empty(n * d, dtype=torch.float32, device="cuda")
    device.synth_prnu(side, side, 0, n, 64, 5, items)
    params = _lib.app_params(_lib.APP_NCC, n, height=side, width=side)
    eng = device.DeviceEngine(params, device_slots=n)
    total = n * (n - 1) // 2
    out = torch.zeros(total, dtype=torch.float64, device="cuda")
    eng.run(out, device_items=items, parsed_stride=d * 4)       # warm-up (preprocess + Gram)
    # time the Gram kernel alone on the resident, normalised slots
    import ctypes as C
    base, stride = C.c_void_p(), C.c_size_t()
    _lib.check(_lib.lib.rk_engine_arena(eng.handle, C.byref(base), C.byref(stride)))
    dapp = device.DeviceApp(params)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        _lib.check(_lib.lib.rk_ncc_gram(dapp.handle, base, stride.value, n, 0, 1, out.data_ptr(), None,
                                        torch.cuda.current_stream().cuda_stream))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tiles = ((n + 127) // 128) * ((n + 127) // 128 + 1) // 2
    flops_tiles = tiles * 2.0 * 128 * 128 * d
    flops_pairs = total * 2.0 * d
    # accuracy: a sample of pairs through the fp32 per-pair path
    rng = np.random.default_rng(0)
    sample = sorted({(int(i), int(j)) for i, j in rng.integers(0, n, size=(256, 2)) if i < j})
    ref = torch.zeros(total, dtype=torch.float64, device="cuda")
    pids = [i * (2 * n - i - 1) // 2 + (j - i - 1) for i, j in sample]
    _lib.check(_lib.lib.rk_compare_pairs(
        dapp.handle, base, stride.value, (_lib.Pair * len(sample))(*[_lib.Pair(i, j, i, j) for i, j in sample]),
        len(sample), ref.data_ptr(), None, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    out_h = out.cpu().numpy()
    g = out_h[pids]
    f = ref.cpu().numpy()[pids]
    print(json.dumps({"n": n, "side": side, "pairs": total, "gram_ms": ms, "pairs_per_s": total / (ms / 1e3),
                      "tf32_tflops_issued": flops_tiles / (ms * 1e-3) / 1e12,
                      "tf32_tflops_useful": flops_pairs / (ms * 1e-3) / 1e12,
                      "max_abs_err_vs_fp32": float(np.max(np.abs(g - f))), "sample": len(sample),
                      "out_sha256": hashlib.sha256(out_h.tobytes()).hexdigest()[:16]}))


if __name__ == "__main__":
    main()
