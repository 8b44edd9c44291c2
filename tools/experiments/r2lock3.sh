# leaf-ordered calibration; ncu captures of job launches (past the calibration launches)
set -x
cd $GRAFT_REPO_ROOT
python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2lock3_1k.log 2>&1
timeout 600 python bench.py --items 512 --side 2048 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2lock3_2k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pce2k_pair -s 14 -c 1 -o gpurun_out/r2lock3_prof_pce2k python bench.py --items 512 --side 2048 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2lock3_ncu_pce2k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pce_cluster -s 14 -c 1 -o gpurun_out/r2lock3_prof_pce python bench.py --items 1024 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2lock3_ncu_pce.log 2>&1
for f in gpurun_out/r2lock3_1k.log gpurun_out/r2lock3_2k.log; do python -c "
import json; l=[x for x in open('$f') if x.startswith('{')]; d=json.loads(l[-1])
print('$f', round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), d['parity']['pass'], d['perf_model'])"; done
