# one 8-warp CTA per SM (2 groups) vs two 4-warp CTAs per SM, each on its own pair
set -x
timeout 600 python -m pytest tests/test_pce_gpu.py -q -x > gpurun_out/grp2_pytest.log 2>&1; echo PYTEST $? >> gpurun_out/grp2_pytest.log
timeout 600 python bench.py --items 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/grp2_a.log 2>&1
RK_NVCC_FLAGS="-DPCE_GROUPS=1" python paper_2009_04755_b200/_build.py --force
timeout 600 python -m pytest tests/test_pce_gpu.py -q -x > gpurun_out/grp1_pytest.log 2>&1; echo PYTEST $? >> gpurun_out/grp1_pytest.log
timeout 600 python bench.py --items 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/grp1_a.log 2>&1
python paper_2009_04755_b200/_build.py --force
timeout 600 python bench.py --items 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/grp2_b.log 2>&1
RK_NVCC_FLAGS="-DPCE_GROUPS=1" python paper_2009_04755_b200/_build.py --force
timeout 600 python bench.py --items 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/grp1_b.log 2>&1
python paper_2009_04755_b200/_build.py --force
