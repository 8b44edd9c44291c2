# split-T timing model (PCE_T16=1: H/L f16x2 planes, row pass reads H only) vs fp32 T, same box
set -x
cd $GRAFT_REPO_ROOT
B="import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
for rep in 1 2; do
for v in 0 1; do
  RK_NVCC_FLAGS="-DPCE_T16=$v" python -c "$B"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2t16a_$v.$rep.log 2>&1
done
done
for rep in 1 2; do for v in 0 1; do python -c "import json; d=json.loads(open('gpurun_out/r2t16a_$v.$rep.log').readline()); print('T16=$v', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done; done
