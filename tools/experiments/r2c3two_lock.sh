# C3 PCE on 2 GPUs with the final kernels (W1 K1)
set -x
cd $GRAFT_REPO_ROOT
python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
timeout 2700 python bench.py --gpus 2 --items 16384 --side 2048 --steps 1 --warmup 1 --no-cpu > gpurun_out/r2c3two_lock.log 2>&1; echo RC $? >> gpurun_out/r2c3two_lock.log
tail -c 300 gpurun_out/r2c3two_lock.log
