set -x
for f in 0 1 0 1; do
  RK_NVCC_FLAGS="-DPCE_PAD_XPOSE=$f" python paper_2009_04755_b200/_build.py --force
  timeout 600 python bench.py --items 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/pad2_$f.log 2>&1
  tail -1 gpurun_out/pad2_$f.log >> gpurun_out/pad2_all.log
done
python paper_2009_04755_b200/_build.py --force
