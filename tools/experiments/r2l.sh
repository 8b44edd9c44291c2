# final 1-GPU evidence with the driver's invocation: tests, smoke, bench (K=20, W=5), reference arm, C5 CV line
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2l_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2l_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1; echo SMOKE $? >> gpurun_out/r2l_smoke.log
/usr/bin/time -v timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2l_bench.log 2> gpurun_out/r2l_bench.err; echo BENCH $? >> gpurun_out/r2l_bench.log
/usr/bin/time -v timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2l_ref.log 2> gpurun_out/r2l_ref.err; echo REF $? >> gpurun_out/r2l_ref.log
timeout 1200 python bench.py --app cv --steps 3 --warmup 3 > gpurun_out/r2l_cv.log 2>&1; echo CV $? >> gpurun_out/r2l_cv.log
tail -2 gpurun_out/r2l_tests.log; tail -2 gpurun_out/r2l_smoke.log; grep "Elapsed" gpurun_out/r2l_bench.err gpurun_out/r2l_ref.err
