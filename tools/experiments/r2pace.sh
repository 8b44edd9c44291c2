# pce2k: grid pacing inside the column phase (RK_PCE_PACE iterations between paces), same box
set -x
cd $GRAFT_REPO_ROOT
python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for rep in 1 2; do
for pc in 0 32 16 8; do
  RK_PCE_PACE=$pc timeout 600 python bench.py --items 512 --side 2048 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2pace_$pc.$rep.log 2>&1
done
done
RK_PCE_PACE=16 timeout 900 ncu --set full --clock-control none -k regex:pce2k_pair -s 2 -c 1 -o gpurun_out/r2pace_prof16 python bench.py --items 300 --side 2048 --steps 1 --warmup 0 --no-e2e --no-cpu --no-parity > gpurun_out/r2pace_ncu.log 2>&1
for f in gpurun_out/r2pace_*.?.log; do python -c "
import json; l=[x for x in open('$f') if x.startswith('{')]; d=json.loads(l[-1])
print('$f', round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), d['parity']['pass'])"; done
