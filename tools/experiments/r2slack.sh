# round barrier slack: start round k when all but s% of the CTAs finished round k-1
set -x
cd $GRAFT_REPO_ROOT
B="import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for v in 0 10 25 0 10 25; do
  RK_NVCC_FLAGS="-DPCE_ROUND_SLACK_PCT=$v" python -c "$B"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2slack_1k_$v.$RANDOM.log 2>&1
  timeout 600 python bench.py --items 512 --side 2048 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2slack_2k_$v.$RANDOM.log 2>&1
done
