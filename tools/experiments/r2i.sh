# 4 GPUs: full GPU suite (multi-GPU test at world 4), C3-Gram with the job breakdown, 1-GPU C2 sanity
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2i_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2i_tests.log
timeout 900 python bench.py --gpus 4 --app ncc --items 16384 --side 2048 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2i_c3ncc.log 2>&1; echo N $? >> gpurun_out/r2i_c3ncc.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2i_c2.log 2>&1; echo B $? >> gpurun_out/r2i_c2.log
tail -3 gpurun_out/r2i_tests.log; tail -c 300 gpurun_out/r2i_c3ncc.log
