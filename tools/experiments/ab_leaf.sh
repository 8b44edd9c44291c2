# leaf size and T store policy A/B (same box)
set -x
for lf in 4 8 12 16; do
  timeout 600 python bench.py --items 2048 --leaf $lf --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/leaf$lf.log 2>&1
done
RK_NVCC_FLAGS="-DPCE_T_POLICY=1" python paper_2009_04755_b200/_build.py --force
timeout 600 python bench.py --items 2048 --leaf 8 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/tfirst.log 2>&1
RK_NVCC_FLAGS="-DPCE_T_POLICY=1 -DPCE_SPEC_POLICY=0" python paper_2009_04755_b200/_build.py --force
timeout 600 python bench.py --items 2048 --leaf 8 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/tfirst_slast.log 2>&1
python paper_2009_04755_b200/_build.py --force
