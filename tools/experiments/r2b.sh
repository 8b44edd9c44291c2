# round 2: GPU tests + TF32 peak + bench lines for ncc / C1 / 2048^2
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/r2b_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2b_tests.log
timeout 300 python tools/tf32_peak.py > gpurun_out/r2b_tf32.json 2> gpurun_out/r2b_tf32.err
cp gpurun_out/r2b_tf32.json profiles/r2_tf32_peak.json 2>/dev/null
timeout 600 python bench.py --app ncc --steps 3 --warmup 3 --no-cpu > gpurun_out/r2b_ncc.log 2>&1; echo NCC $? >> gpurun_out/r2b_ncc.log
timeout 600 python bench.py --items 128 --side 256 --steps 5 --warmup 3 > gpurun_out/r2b_c1.log 2>&1; echo C1 $? >> gpurun_out/r2b_c1.log
timeout 900 python bench.py --items 512 --side 2048 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2b_2k.log 2>&1; echo 2K $? >> gpurun_out/r2b_2k.log
tail -3 gpurun_out/r2b_tests.log
