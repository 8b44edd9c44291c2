# round barrier defaults: 2048^2 leaf 8 / 16, 1024^2 headline, ncu of both compare kernels, GPU tests
set -x
cd $GRAFT_REPO_ROOT
python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for lf in 8 16; do
  timeout 600 python bench.py --items 512 --side 2048 --leaf $lf --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2lock2_2k_leaf$lf.log 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2lock2_1k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pce2k_pair -s 2 -c 1 -o gpurun_out/r2lock2_prof_pce2k python bench.py --items 300 --side 2048 --steps 1 --warmup 0 --no-e2e --no-cpu --no-parity > gpurun_out/r2lock2_ncu_pce2k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pce_cluster -s 2 -c 1 -o gpurun_out/r2lock2_prof_pce python bench.py --items 1024 --steps 1 --warmup 0 --no-e2e --no-cpu --no-parity > gpurun_out/r2lock2_ncu_pce.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2lock2_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2lock2_tests.log
for f in gpurun_out/r2lock2_*k*.log; do python -c "
import json; l=[x for x in open('$f') if x.startswith('{')]; d=json.loads(l[-1]) if l else None
print('$f', d and (round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), d.get('parity',{}).get('pass')))"; done
tail -3 gpurun_out/r2lock2_tests.log
