# refill fences on (old) vs off (new), same box; 1024^2 and 2048^2
set -x
for f in 1 0; do
  RK_NVCC_FLAGS="-DPCE_REFILL_FENCE=$f" python paper_2009_04755_b200/_build.py --force
  timeout 600 python bench.py --items 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/fence$f.log 2>&1
  timeout 600 python bench.py --items 384 --side 2048 --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/fence${f}_2k.log 2>&1
done
python paper_2009_04755_b200/_build.py --force
timeout 900 python -m pytest tests/test_pce_gpu.py tests/test_peer_tier_gpu.py -q -x > gpurun_out/fence_pytest.log 2>&1; echo PYTEST $? >> gpurun_out/fence_pytest.log
