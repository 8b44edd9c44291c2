"""Per-phase clock breakdown of pce_cluster (librocket built with -DPCE_PROBES)."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2009_04755_b200 import _lib, device
n, side = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 1024
items = torch.empty(n * side * side, dtype=torch.float32, device="cuda")
device.synth_prnu(side, side, 0, n, 4, 1, items)
eng = device.DeviceEngine(_lib.app_params(_lib.APP_PCE, n, height=side, width=side), leaf_block=8, device_slots=n)
out = torch.zeros(n * (n - 1) // 2, dtype=torch.float64, device="cuda")
eng.run(out, device_items=items, parsed_stride=side * side * 4)
buf = (C.c_ulonglong * (148 * 2 * 8))()
_lib.lib.rk_debug_pce_probes(buf, 148 * 2 * 8, 1)
eng.run(out, device_items=items, parsed_stride=side * side * 4)
torch.cuda.synchronize()
_lib.lib.rk_debug_pce_probes(buf, 148 * 2 * 8, 0)
a = np.array(buf, dtype=np.float64).reshape(148, 2, 8)
pairs = n * (n - 1) // 2
used = a[:, 0, 0] > 0
ctas = used.sum()
cl = int(sys.argv[2]) if len(sys.argv) > 2 else 1
clusters = ctas // cl
per_cluster_pairs = pairs / clusters
names = ["column", "barrier1", "row", "reduce+barrier2", "window", "barrier3", "(next pair)"]
for w in range(2):
    d = np.diff(a[used, w, :7], axis=1) / per_cluster_pairs  # clocks per pair per phase
    print("warp", 0 if w == 0 else 15, " ".join(f"{nm}={v:.0f}" for nm, v in zip(names, d.mean(0))))
print("ctas", ctas, "pairs", pairs)
