# NCC Gram with the interleaved slot layout: tests, then K-chunk size per launch (same box)
set -x
timeout 300 python -m pytest tests/test_ncc_gpu.py -q -x > gpurun_out/kc_pytest.log 2>&1; echo PYTEST $? >> gpurun_out/kc_pytest.log
for kc in 2048 32768; do
  RK_NVCC_FLAGS="-DNCC_KCHUNK=$kc" python paper_2009_04755_b200/_build.py --force
  timeout 300 python tools/ncc_bench.py 4096 1024 > gpurun_out/kc_$kc.log 2>&1
done
python paper_2009_04755_b200/_build.py --force
