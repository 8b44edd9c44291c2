# C3 PCE on 4 GPUs with the contract's warm-up (W = 3, K = 1)
set -x
cd $GRAFT_REPO_ROOT
timeout 4000 python bench.py --gpus 4 --items 16384 --side 2048 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2u_c3pce.log 2>&1; echo P $? >> gpurun_out/r2u_c3pce.log
tail -c 600 gpurun_out/r2u_c3pce.log
