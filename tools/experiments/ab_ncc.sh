# NCC Gram: parity tests of the CTA-pair kernel, then the 128-tile kernel (4 / 6 stages) vs the pair kernel
set -x
timeout 300 python -m pytest tests/test_ncc_gpu.py -q -x > gpurun_out/ncc_pytest.log 2>&1; echo PYTEST $? >> gpurun_out/ncc_pytest.log
timeout 300 python tools/ncc_bench.py 4096 1024 > gpurun_out/ncc_pair.log 2>&1
for st in 4 6; do
  RK_NVCC_FLAGS="-DNCC_STAGES=$st -DNCC_GRAM_1CTA" python paper_2009_04755_b200/_build.py --force
  timeout 300 python tools/ncc_bench.py 4096 1024 > gpurun_out/ncc_1cta_st$st.log 2>&1
done
python paper_2009_04755_b200/_build.py --force
