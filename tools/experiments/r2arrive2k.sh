# pce2k row phase: counted-arrival half release (PCE2K_ROW_ARRIVE=1) vs the group barrier (0), same box
set -x
cd $GRAFT_REPO_ROOT
B="import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for rep in 1 2; do
for v in 0 1; do
  RK_NVCC_FLAGS="-DPCE2K_ROW_ARRIVE=$v" python -c "$B"
  timeout 600 python bench.py --items 512 --side 2048 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2arrive2k_$v.$rep.log 2>&1
done
done
RK_NVCC_FLAGS="-DPCE2K_ROW_ARRIVE=1" python -c "$B"
timeout 600 python tools/pce_determinism.py --side 2048 --n 24 --runs 5 > gpurun_out/r2arrive2k_det.log 2>&1
timeout 900 python -m pytest tests/test_pce_gpu.py -q > gpurun_out/r2arrive2k_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2arrive2k_tests.log
