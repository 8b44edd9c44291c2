# determinism of the PCE path at 256^2 / 1024^2, default build vs refill proxy fences; NCC peer tests
set -x
cd $GRAFT_REPO_ROOT
for cfg in "--side 256 --n 72 --runs 4" "--side 256 --n 24 --runs 6 --leaf 4 --slots 6" "--side 1024 --n 40 --runs 3"; do
  timeout 300 python tools/pce_determinism.py $cfg >> gpurun_out/r2c_det_default.log 2>&1
done
timeout 600 python -m pytest tests/test_peer_tier_gpu.py -q -k ncc > gpurun_out/r2c_ncc.log 2>&1; echo NCC $? >> gpurun_out/r2c_ncc.log
RK_NVCC_FLAGS="-DPCE_REFILL_FENCE=1" python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for cfg in "--side 256 --n 72 --runs 4" "--side 256 --n 24 --runs 6 --leaf 4 --slots 6"; do
  timeout 300 python tools/pce_determinism.py $cfg >> gpurun_out/r2c_det_fence.log 2>&1
done
cat gpurun_out/r2c_det_default.log gpurun_out/r2c_det_fence.log | cut -c 1-600
tail -3 gpurun_out/r2c_ncc.log
