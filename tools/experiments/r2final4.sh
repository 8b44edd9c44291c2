# final 4-GPU box regression with the round-barrier kernels: GPU tests, C2 on 1 / 4 GPUs
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2final4_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2final4_smoke.log 2>&1; echo SMOKE $? >> gpurun_out/r2final4_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2final4_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2final4_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2final4_c2_1gpu.log 2>&1
timeout 900 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/r2final4_c2_4gpu.log 2>&1
tail -2 gpurun_out/r2final4_smoke.log; tail -3 gpurun_out/r2final4_tests.log
for f in gpurun_out/r2final4_c2_*.log; do python -c "
import json; l=[x for x in open('$f') if x.startswith('{')]; d=json.loads(l[-1])
print('$f', round(d['value']), d['e2e']['value'], d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), d['parity']['pass'], d['ledger']['full'], d['perf_model']['efficiency'])"; done
