# refill-fence variants: determinism (many runs) and bench throughput at C2
set -x
cd $GRAFT_REPO_ROOT
for v in 1 2 0; do
  RK_NVCC_FLAGS="-DPCE_REFILL_FENCE=$v" python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
  timeout 300 python tools/pce_determinism.py --side 256 --n 72 --runs 10 > gpurun_out/r2d_det_f$v.log 2>&1
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-parity > gpurun_out/r2d_bench_f$v.log 2>&1
done
python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2d_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2d_tests.log
for v in 1 2 0; do cut -c 1-300 gpurun_out/r2d_det_f$v.log; python -c "import json; d=json.loads(open('gpurun_out/r2d_bench_f$v.log').readline()); print('f$v', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
tail -3 gpurun_out/r2d_tests.log
