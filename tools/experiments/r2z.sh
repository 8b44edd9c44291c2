# final state: GPU suite, smoke, default bench line
set -x
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2z_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2z_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; echo SMOKE $? >> gpurun_out/r2z_smoke.log
timeout 1200 python bench.py > gpurun_out/r2z_bench.log 2>&1; echo BENCH $? >> gpurun_out/r2z_bench.log
tail -2 gpurun_out/r2z_tests.log; tail -1 gpurun_out/r2z_smoke.log; tail -c 400 gpurun_out/r2z_bench.log
