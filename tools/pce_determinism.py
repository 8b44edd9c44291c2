"""Run-to-run determinism of the PCE compare path (diagnostic).

The same all-pairs job is run several times through the engine (fixed leaf and
slot tier, so the same pairs land in the same launches); every run must be
bit-identical.  Mismatching pair ids are recomputed by the float64 oracle to
show which run is wrong.  Prints one JSON line.

  python tools/pce_determinism.py --side 256 --n 72 --runs 4
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--n", type=int, default=72)
    ap.add_argument("--runs", type=int, default=4)
    ap.add_argument("--leaf", type=int, default=8)
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--cameras", type=int, default=6)
    ap.add_argument("--seed", type=int, default=17)
    args = ap.parse_args()
    from oracle import pce as opce
    from oracle import scheduler as osch
    from paper_2009_04755_b200 import _lib, device
    n, side = args.n, args.side
    items = torch.empty(n * side * side, dtype=torch.float32, device="cuda")
    device.synth_prnu(side, side, 0, n, args.cameras, args.seed, items)
    total = n * (n - 1) // 2
    outs = []
    for _ in range(args.runs):
        eng = device.DeviceEngine(_lib.app_params(_lib.APP_PCE, n, height=side, width=side, threshold=60.0),
                                  leaf_block=args.leaf, device_slots=args.slots or n)
        out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
        eng.run(out, device_items=items, parsed_stride=side * side * 4)
        outs.append(out.cpu().numpy())
        eng.close()
    stack = np.stack(outs)
    bad = np.flatnonzero(np.any(stack != stack[0], axis=0))
    rep = {"side": side, "n": n, "pairs": total, "runs": args.runs, "mismatching_pids": int(len(bad))}
    if len(bad):
        host = items.cpu().numpy().reshape(n, side, side)
        sample = bad[:16].tolist()
        pairs = [osch.pair_from_id(n, p) for p in sample]
        want = opce.pairs_batched(host, pairs, batch=4)
        rep["detail"] = [{"pid": p, "pair": pr, "oracle": float(w), "runs": stack[:, p].tolist(),
                          "run_rel_err": (np.abs(stack[:, p] - w) / abs(w)).tolist()}
                         for p, pr, w in zip(sample, pairs, want)]
    # and every run against the oracle (all pairs for small jobs)
    if total <= 4096:
        host = items.cpu().numpy().reshape(n, side, side)
        want = opce.pairs_batched(host, [osch.pair_from_id(n, p) for p in range(total)])
        rel = np.abs(stack - want[None, :]) / np.abs(want)[None, :]
        rep["max_rel_err_per_run"] = rel.max(axis=1).tolist()
        rep["pairs_over_1e-5_per_run"] = (rel > 1e-5).sum(axis=1).tolist()
    print(json.dumps(rep), flush=True)


if __name__ == "__main__":
    main()
