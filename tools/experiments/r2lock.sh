# PCE compare grids: round barrier (RK_PCE_LOCKSTEP) and L2 policies (RK_PCE_L2OPTS), same box, interleaved
set -x
cd $GRAFT_REPO_ROOT
python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for rep in 1 2; do
for v in "0 0" "1 0" "1 1" "1 3"; do
  set -- $v
  RK_PCE_LOCKSTEP=$1 RK_PCE_L2OPTS=$2 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2lock_1k_$1$2.$rep.log 2>&1
done
done
for v in "0 0" "1 0" "1 1" "1 3"; do
  set -- $v
  RK_PCE_LOCKSTEP=$1 RK_PCE_L2OPTS=$2 timeout 600 python bench.py --items 512 --side 2048 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2lock_2k_$1$2.log 2>&1
done
for f in gpurun_out/r2lock_*.log; do python -c "
import json; l=[x for x in open('$f') if x.startswith('{')]; d=json.loads(l[-1])
print('$f', round(d['value']), d['clocks']['sm_mhz'], d['roofline']['frac'], d.get('parity',{}).get('pass'))"; done
