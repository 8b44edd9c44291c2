# final 1-GPU evidence with the driver's invocation: tests, smoke, bench (K=20, W=5), reference arm, C5 CV line
set -x
cd $GRAFT_REPO_ROOT
t0=$(date +%s); timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2l_bench.log 2> gpurun_out/r2l_bench.err; echo BENCH $? >> gpurun_out/r2l_bench.log; echo bench_s $(( $(date +%s) - t0 )) >> gpurun_out/r2l_times.txt
t0=$(date +%s); timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2l_ref.log 2> gpurun_out/r2l_ref.err; echo REF $? >> gpurun_out/r2l_ref.log; echo ref_s $(( $(date +%s) - t0 )) >> gpurun_out/r2l_times.txt
tail -2 gpurun_out/r2l_tests.log; tail -2 gpurun_out/r2l_smoke.log; cat gpurun_out/r2l_times.txt
