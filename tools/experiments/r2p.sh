# CV: 32-bit key fast path (new) vs 64-bit shuffles (old): CV tests + A/B on the C5 line
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_apps_gpu.py tests/test_dropin_gpu.py -q > gpurun_out/r2p_tests.log 2>&1; echo T $? >> gpurun_out/r2p_tests.log
cp paper_2009_04755_b200/csrc/cv.cu /tmp/cv_new.cu
for v in new old new; do
  if [ $v = old ]; then cp tools/experiments/ab_old/cv.cu paper_2009_04755_b200/csrc/cv.cu; else cp /tmp/cv_new.cu paper_2009_04755_b200/csrc/cv.cu; fi
  python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
  timeout 900 python bench.py --app cv --steps 3 --warmup 2 --no-cpu --no-e2e >> gpurun_out/r2p_cv_$v.log 2>&1
done
tail -2 gpurun_out/r2p_tests.log
for v in new old; do python -c "
import json
for l in open('gpurun_out/r2p_cv_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['ms_per_step'])"; done
