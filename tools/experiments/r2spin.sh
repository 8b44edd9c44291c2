# round-barrier spin limit (cycles) at 2048^2 and 1024^2
set -x
cd $GRAFT_REPO_ROOT
B="import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for v in 200000 2000000 50000 200000 2000000; do
  RK_NVCC_FLAGS="-DPCE_ROUND_SPIN=$v" python -c "$B"
  timeout 600 python bench.py --items 512 --side 2048 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2spin_2k_$v.$RANDOM.log 2>&1
done
