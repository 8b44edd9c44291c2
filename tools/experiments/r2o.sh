# GMM: angle pairs on the FMA-pipe polynomial exp2 (0 / 1 / 2 of 6), C4 line
set -x
cd $GRAFT_REPO_ROOT
for v in 1 0 2 1; do
  RK_NVCC_FLAGS="-DGMM_POLY_PAIRS=$v" python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
  timeout 600 python -m pytest tests/test_gmm_gpu.py -q >> gpurun_out/r2o_tests.log 2>&1
  timeout 600 python bench.py --app gmm --steps 5 --warmup 3 --no-cpu --no-e2e >> gpurun_out/r2o_gmm_$v.log 2>&1
done
grep -c passed gpurun_out/r2o_tests.log; grep failed gpurun_out/r2o_tests.log
for v in 0 1 2; do python -c "
import json
for l in open('gpurun_out/r2o_gmm_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['ms_per_step'])"; done
