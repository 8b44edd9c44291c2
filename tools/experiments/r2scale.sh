# C2 scaling on one 4-GPU box, back to back (the driver's SCALE protocol at N = 1, 2, 4)
set -x
cd $GRAFT_REPO_ROOT
for g in 1 2 4; do
  timeout 1500 python bench.py --gpus $g --steps 3 --warmup 3 --no-cpu > gpurun_out/r2scale_$g.log 2>&1
done
for g in 1 2 4; do python -c "
import json
for l in open('gpurun_out/r2scale_$g.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$g', round(d['value']), round(d['e2e']['value']), d['clocks']['sm_mhz'], d['perf_model']['efficiency'], d['parity']['pass'], d['ledger']['full'])"; done
