set -x
for pp in 0 2 3; do
  RK_NVCC_FLAGS="-DGMM_POLY=$pp" python paper_2009_04755_b200/_build.py --force
  RK_NO_CLOCKS=1 timeout 300 python bench.py --app gmm --no-e2e --no-cpu > gpurun_out/poly$pp.log 2>&1
done
python paper_2009_04755_b200/_build.py --force
