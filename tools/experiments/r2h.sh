# A/B: padded vs XOR-swizzled transpose in pce_cluster (C2 bench), determinism; host memory size
set -x
cd $GRAFT_REPO_ROOT
free -g > gpurun_out/r2h_free.txt; nproc >> gpurun_out/r2h_free.txt
for v in 1 0 1; do
  RK_NVCC_FLAGS="-DPCE_XPOSE_PAD=$v" python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-parity >> gpurun_out/r2h_bench_pad$v.log 2>&1
done
timeout 300 python tools/pce_determinism.py --side 256 --n 72 --runs 6 > gpurun_out/r2h_det.log 2>&1
timeout 300 python tools/pce_determinism.py --side 1024 --n 64 --runs 2 >> gpurun_out/r2h_det.log 2>&1
for v in 1 0; do for l in $(grep -c . gpurun_out/r2h_bench_pad$v.log); do :; done; python -c "
import json
for l in open('gpurun_out/r2h_bench_pad$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('pad$v', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
cut -c 1-300 gpurun_out/r2h_det.log; cat gpurun_out/r2h_free.txt
