# 1024^2 headline: round barrier off / on, same box, three interleaved reps
set -x
cd $GRAFT_REPO_ROOT
python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for rep in 1 2 3; do
for v in 0 1; do
  RK_PCE_LOCKSTEP=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2lock4_$v.$rep.log 2>&1
done
done
