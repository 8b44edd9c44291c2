# A/B: row-pair argmax tracking + locate step (new) vs per-element index search (old)
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_pce_gpu.py tests/test_ledger_gpu.py -q -x > gpurun_out/r2k_tests.log 2>&1; echo T $? >> gpurun_out/r2k_tests.log
timeout 300 python tools/pce_determinism.py --side 256 --n 72 --runs 4 > gpurun_out/r2k_det.log 2>&1
for v in new old new old; do
  if [ $v = old ]; then cp tools/experiments/ab_old/pce.cu paper_2009_04755_b200/csrc/pce.cu; cp tools/experiments/ab_old/pce_common.cuh paper_2009_04755_b200/csrc/pce_common.cuh; fi
  if [ $v = new ]; then cp gpurun_out/../paper_2009_04755_b200/csrc/pce.cu /dev/null; fi
  python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-parity >> gpurun_out/r2k_bench_$v.log 2>&1
  if [ $v = old ]; then cp /tmp/new_pce.cu paper_2009_04755_b200/csrc/pce.cu; cp /tmp/new_common.cuh paper_2009_04755_b200/csrc/pce_common.cuh; fi
  if [ $v = new ]; then cp paper_2009_04755_b200/csrc/pce.cu /tmp/new_pce.cu; cp paper_2009_04755_b200/csrc/pce_common.cuh /tmp/new_common.cuh; fi
done
tail -2 gpurun_out/r2k_tests.log; cut -c 1-160 gpurun_out/r2k_det.log
for v in new old; do python -c "
import json
for l in open('gpurun_out/r2k_bench_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],1))"; done
