"""Timeline diagnosis of an engine run from its trace events: span, busy time per
lane and the largest idle gaps between consecutive compare batches.

  python tools/gap_trace.py gmm|cv [--items N] [--runs R]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2009_04755_b200 import _lib, device, synthdata  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("app", choices=["gmm", "cv", "pce"])
    ap.add_argument("--items", type=int, default=0)
    ap.add_argument("--runs", type=int, default=4)
    a = ap.parse_args()
    if a.app == "gmm":
        n = a.items or 1000
        host, _ = synthdata.gmm_parsed(n, 1, 400)
        stride = host.shape[1]
        items = torch.from_numpy(host.reshape(-1)).cuda()
        params = _lib.app_params(_lib.APP_GMM, n, max_entries=400, gmm_angles=36)
    elif a.app == "pce":
        n, side = a.items or 1024, 1024
        items = torch.empty(n * side * side, dtype=torch.float32, device="cuda")
        device.synth_prnu(side, side, 0, n, 64, 1, items)
        stride = side * side * 4
        params = _lib.app_params(_lib.APP_PCE, n, height=side, width=side, threshold=60.0)
    else:
        n = a.items or 600
        items, stride, cap, _ = synthdata.cv_parsed_device(n, 5e5, 1)
        params = _lib.app_params(_lib.APP_CV, n, max_entries=cap)
    eng = device.DeviceEngine(params, leaf_block=8 if a.app == "pce" else 16, device_slots=n)
    eng.set_trace(100000)
    out = torch.zeros(n * (n - 1) // 2, dtype=torch.float64, device="cuda")
    for r in range(a.runs):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.run(out, device_items=items, parsed_stride=stride)
        e1.record()
        torch.cuda.synchronize()
        ev = eng.trace()
        comp = sorted([e for e in ev if e["label"] == "compare"], key=lambda e: e["start_ns"])
        loads = [e for e in ev if e["label"] != "compare"]
        span = max(e["end_ns"] for e in ev) - min(e["start_ns"] for e in ev)
        busy = sum(e["end_ns"] - e["start_ns"] for e in comp)
        gaps = sorted(((comp[k + 1]["start_ns"] - comp[k]["end_ns"], k) for k in range(len(comp) - 1)), reverse=True)
        print(json.dumps({"run": r, "wall_ms": e0.elapsed_time(e1), "span_ms": span / 1e6,
                          "compare_busy_ms": busy / 1e6, "compare_batches": len(comp),
                          "load_busy_ms": sum(e["end_ns"] - e["start_ns"] for e in loads) / 1e6,
                          "load_groups": len(loads),
                          "top_gaps_ms": [round(g / 1e6, 3) for g, _ in gaps[:8]],
                          "median_batch_ms": sorted(e["end_ns"] - e["start_ns"] for e in comp)[len(comp) // 2] / 1e6}))


if __name__ == "__main__":
    main()
