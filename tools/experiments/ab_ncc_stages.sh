# NCC Gram (CTA pair): K chunk per launch 1024 / 2048 / 4096 k-blocks and 6 vs 7 pipeline stages (same box)
mkdir -p gpurun_out
CFGS=${NCC_CFGS:-"2048:6 1024:6 4096:6 2048:7 2048:6"}
for cfg in $CFGS; do
  set -- ${cfg/:/ }
  RK_NVCC_FLAGS="-DNCC_KCHUNK=$1 -DNCC_STAGES=$2" python paper_2009_04755_b200/_build.py --force > /dev/null 2>&1
  echo "kchunk=$1 stages=$2 $(timeout 300 python tools/ncc_bench.py 4096 1024 2>&1 | tail -1)"
done
python paper_2009_04755_b200/_build.py --force > /dev/null 2>&1
timeout 300 python -m pytest tests/test_ncc_gpu.py -q -x 2>&1 | tail -1
