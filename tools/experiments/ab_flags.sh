# Same-box A/B of two librocket build-flag sets on the C2 bench (N = 2,048 subset):
#   bash tools/experiments/ab_flags.sh "<flags A>" "<flags B>" [tag]
# runs the PCE GPU tests on B, then A B A B bench lines; leaves the default build.
A="$1"; B="$2"; T="${3:-ab}"
b() { RK_NVCC_FLAGS="$1" python paper_2009_04755_b200/_build.py --force > /dev/null; }
b "$B"; timeout 600 python -m pytest tests/test_pce_gpu.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo PYTEST $? >> gpurun_out/${T}_pytest.log
for r in 1 2; do
  for v in A B; do
    if [ $v = A ]; then b "$A"; else b "$B"; fi
    timeout 600 python bench.py ${BENCH_ARGS:---items 2048} --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_${v}${r}.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/${T}_${v}${r}.log').read().strip().splitlines()[-1]); print('$v$r', round(d['value']), d['roofline']['ms_per_launch'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" | tee -a gpurun_out/${T}_summary.log
  done
done
tail -1 gpurun_out/${T}_pytest.log
python paper_2009_04755_b200/_build.py --force > /dev/null
