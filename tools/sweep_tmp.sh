for cfg in "1 2 2 8" "2 2 2 16" "2 2 0 8" "2 2 2 4" "4 2 2 8"; do
  set -- $cfg
  RK_NVCC_FLAGS="-DPCE_CL=$1 -DPCE_T_POLICY=$2 -DPCE_SPEC_POLICY=$3" python paper_2009_04755_b200/_build.py --force >/dev/null
  python bench.py --n 1024 --leaf $4 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/sw2_$1_$2_$3_$4.log 2>&1
done
