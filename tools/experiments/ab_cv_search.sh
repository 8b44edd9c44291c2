# A/B (not kept: 253k vs 277k pairs/s; the source no longer has the switch) of the CV merge's B-window binary search: shared memory (CV_SMEM_SEARCH=1, the
# in-tree build) vs 64-bit shuffles (rebuilt with -DCV_SMEM_SEARCH=0), C5 via bench.py --app cv
mkdir -p gpurun_out
python -m pytest tests/test_apps_gpu.py -q -x -k cv 2>&1 | tail -1
for r in 1 2; do
  python bench.py --app cv --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('smem', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
RK_NVCC_FLAGS=-DCV_SMEM_SEARCH=0 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -m pytest tests/test_apps_gpu.py -q -x -k cv 2>&1 | tail -1
for r in 1 2; do
  python bench.py --app cv --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('shfl', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
