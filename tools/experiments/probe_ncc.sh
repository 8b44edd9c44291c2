# NCC Gram pair kernel: feed-only and MMA-only probes (diagnostic builds)
set -x
for f in NCC_PROBE_NOTMA NCC_PROBE_NOMMA; do
  RK_NVCC_FLAGS="-D$f" python paper_2009_04755_b200/_build.py --force
  timeout 300 python tools/ncc_bench.py 4096 1024 > gpurun_out/probe_$f.log 2>&1
done
python paper_2009_04755_b200/_build.py --force
