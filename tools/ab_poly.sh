set -x
for pp in 0 2 3 4; do
  RK_NVCC_FLAGS="-DGMM_POLY=$pp" python paper_2009_04755_b200/_build.py --force
  RK_NO_CLOCKS=1 timeout 300 python bench.py --app gmm --no-e2e --no-cpu > gpurun_out/poly$pp.log 2>&1
done
python paper_2009_04755_b200/_build.py --force
timeout 300 python -m pytest tests/test_gmm_gpu.py -q > gpurun_out/poly_pytest.log 2>&1; echo PYTEST $? >> gpurun_out/poly_pytest.log
