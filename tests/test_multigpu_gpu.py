"""Real multi-GPU runs (one process per GPU, NCCL): results identical bit for bit
to a single-GPU run and every pair written exactly once, with the peer tier and
cross-GPU stealing active.  Needs >= 2 visible GPUs (skipped otherwise)."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_multi_gpu_bit_exact_vs_single_gpu():
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(ngpu, 4)
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", os.path.join(here, "_mgpu_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [l for l in p.stdout.splitlines() if l.startswith("MGPU_REPORT ")]
    assert line, p.stdout[-2000:]
    r = json.loads(line[-1][len("MGPU_REPORT "):])
    assert r["world"] == world and r["pce_pairs"] == 40 * 39 // 2
    assert r["pce_max_rel_err"] <= 1e-4
    assert r["pce_bit_exact_vs_1gpu"] and r["pce_flags_once"]
    assert r["cv_bit_exact_vs_1gpu"] and r["cv_flags_once"]
    assert r["peer_fetches"] > 0
    assert r["pce_ledger_full"] and r["cv_ledger_full"]          # the shared device ledger on rank 0
