set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2a_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2a_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2a_bench.log 2>&1; echo BENCH $? >> gpurun_out/r2a_bench.log
timeout 300 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2a_ref.log 2>&1; echo REF $? >> gpurun_out/r2a_ref.log
tail -5 gpurun_out/r2a_tests.log; tail -c 3000 gpurun_out/r2a_bench.log
