# flakiness check of the multi-process GPU tests and the determinism test
set -x
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_peer_tier_gpu.py tests/test_dropin_gpu.py tests/test_ledger_gpu.py "tests/test_pce_gpu.py::test_compare_is_deterministic_run_to_run" -q -p no:randomly > gpurun_out/r2flaky_$i.log 2>&1; tail -1 gpurun_out/r2flaky_$i.log
done
