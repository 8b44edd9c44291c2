"""bench.py's driver contract on CPU: the reference arm's JSON line (keys, measured
step time, same config dict as the GPU arm) and the launch checks of --gpus."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=ROOT)


def test_reference_arm_line_keeps_the_contract():
    p = _run(["--impl", "reference", "--items", "64", "--side", "256", "--steps", "2", "--warmup", "1",
              "--cpu-seconds", "2"])
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["value"] > 0 and line["extrapolated"] is False
    assert line["ms_per_step"] == sum(line["cpu_baseline"]["step_ms"]) / 2      # measured, not extrapolated
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    # the GPU arm builds its config with the same function: identical dicts at the same N
    sys.path.insert(0, ROOT)
    import bench
    args = bench.parse_args(["--items", "64", "--side", "256"])
    assert line["config"] == bench.workload(args, 1)[1]
    # the reference's own RealEngine harness on a bounded sample, when oracle/_ref is staged
    re_ = line.get("realengine")
    if isinstance(re_, list):
        assert all(r["ledger_full"] and r["value"] > 0 for r in re_)


def test_world_size_must_match_gpus():
    p = _run(["--gpus", "1"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}, timeout=120)
    assert p.returncode == 2 and "WORLD_SIZE" in p.stderr


def test_calibration_pairs_cover_the_triangle_once_in_leaf_order():
    """The perf-model calibration lists every pair of its items exactly once, in
    the engine's leaf order: leaf x leaf blocks, a block's pairs contiguous."""
    sys.path.insert(0, ROOT)
    import bench
    for m, leaf in ((64, 8), (64, 16), (37, 8), (10, 3), (5, 1)):
        pairs = bench.leaf_ordered_pairs(m, leaf)
        assert len(pairs) == len(set(pairs)) == m * (m - 1) // 2
        assert all(0 <= i < j < m for i, j in pairs)
        blocks = [(i // leaf, j // leaf) for i, j in pairs]
        runs = [b for k, b in enumerate(blocks) if k == 0 or b != blocks[k - 1]]
        assert len(runs) == len(set(runs))      # each block appears as one contiguous run
