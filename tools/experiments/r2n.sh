# GMM: FMA-pipe reciprocal (new) vs MUFU.RCP (old, packed loop both): tests + A/B on the C4 line
set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gmm_gpu.py -q > gpurun_out/r2n_tests.log 2>&1; echo T $? >> gpurun_out/r2n_tests.log
cp paper_2009_04755_b200/csrc/gmm.cu /tmp/gmm_new.cu
for v in new old new old; do
  if [ $v = old ]; then cp tools/experiments/ab_old/gmm.cu paper_2009_04755_b200/csrc/gmm.cu; else cp /tmp/gmm_new.cu paper_2009_04755_b200/csrc/gmm.cu; fi
  python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
  timeout 600 python bench.py --app gmm --steps 5 --warmup 3 --no-cpu --no-e2e >> gpurun_out/r2n_gmm_$v.log 2>&1
done
tail -2 gpurun_out/r2n_tests.log
for v in new old; do python -c "
import json
for l in open('gpurun_out/r2n_gmm_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done
