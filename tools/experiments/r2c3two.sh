# C3 PCE on 2 GPUs (128 GiB of home spectra per GPU), W = 1, K = 1: the 2-GPU point of the C3 curve
set -x
cd $GRAFT_REPO_ROOT
timeout 5000 python bench.py --gpus 2 --items 16384 --side 2048 --steps 1 --warmup 1 --no-cpu > gpurun_out/r2c3two.log 2>&1; echo P $? >> gpurun_out/r2c3two.log
tail -c 400 gpurun_out/r2c3two.log
