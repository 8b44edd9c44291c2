# A/B of the 2048^2 compare kernel variants on one box (same GPU, back to back)
set -x
python paper_2009_04755_b200/_build.py --force
timeout 600 python bench.py --items 512 --side 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab2k_rt.log 2>&1
RK_NVCC_FLAGS=-DPCE2K_SMEM_TW python paper_2009_04755_b200/_build.py --force
timeout 600 python bench.py --items 512 --side 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab2k_smem.log 2>&1
python paper_2009_04755_b200/_build.py --force
timeout 600 python -m pytest tests/test_pce_gpu.py -q -x -k 2048 > gpurun_out/ab2k_pytest.log 2>&1
