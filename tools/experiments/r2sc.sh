# C5 CV on 4 GPUs: work-queue grab size (0 = one 1,024-pair batch = 4 leaves, 1 leaf, 2 leaves)
set -x
cd $GRAFT_REPO_ROOT
for c in 0 1 2; do
  timeout 900 python bench.py --gpus 4 --app cv --steps 3 --warmup 2 --no-cpu --no-e2e --steal-chunk $c > gpurun_out/r2sc_cv4_c$c.log 2>&1
done
for c in 0 1 2; do python -c "
import json
for l in open('gpurun_out/r2sc_cv4_c$c.log'):
    if l.startswith('{'):
        d=json.loads(l); print('c$c', round(d['value']), d['ms_per_step'], d['cache'])"; done
