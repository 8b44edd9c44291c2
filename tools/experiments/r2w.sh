set -x
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --gpus 4 --app ncc --steps 3 --warmup 3 --no-cpu > gpurun_out/r2w_ncc4.log 2>&1
timeout 900 python bench.py --gpus 2 --app ncc --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2w_ncc2.log 2>&1
timeout 900 python -m pytest tests/test_peer_tier_gpu.py tests/test_multigpu_gpu.py tests/test_ncc_gpu.py -q > gpurun_out/r2w_tests.log 2>&1
tail -2 gpurun_out/r2w_tests.log
