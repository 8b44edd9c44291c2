# full regression on one GPU: tests, smoke, bench (N=1 default)
set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r1f_pytest.log 2>&1; echo PYTEST $? >> gpurun_out/r1f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r1f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r1f_bench.log 2>&1; echo BENCH $? >> gpurun_out/r1f_bench.log
