set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --gpus 2 --app ncc --items 16384 --side 2048 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2c3ncc2.log 2>&1; echo N $? >> gpurun_out/r2c3ncc2.log
tail -c 300 gpurun_out/r2c3ncc2.log
