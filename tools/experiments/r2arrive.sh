# PCE row phase: counted-arrival buffer release (PCE_ROW_ARRIVE=1) vs the group barrier (0), same box
set -x
cd $GRAFT_REPO_ROOT
B="import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for rep in 1 2; do
for v in 0 1; do
  RK_NVCC_FLAGS="-DPCE_ROW_ARRIVE=$v" python -c "$B"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2arrive_$v.$rep.log 2>&1
done
done
RK_NVCC_FLAGS="-DPCE_ROW_ARRIVE=1" python -c "$B"
timeout 300 python tools/pce_determinism.py --side 256 --n 72 --runs 10 > gpurun_out/r2arrive_det.log 2>&1
timeout 900 python -m pytest tests/test_pce_gpu.py tests/test_apps_gpu.py -q > gpurun_out/r2arrive_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2arrive_tests.log
for f in gpurun_out/r2arrive_?.?.log; do python -c "
import json; l=[x for x in open('$f') if x.startswith('{')]; d=json.loads(l[-1])
print('$f', round(d['value']), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],1), d['roofline']['ms_per_launch'])"; done
tail -2 gpurun_out/r2arrive_det.log; tail -2 gpurun_out/r2arrive_tests.log
