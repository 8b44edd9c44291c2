# NCC preprocess in L2-sized chunks (new) vs 64-item chunks (old): C2 NCC line A/B + NCC tests
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_ncc_gpu.py -q > gpurun_out/r2x_tests.log 2>&1
cp paper_2009_04755_b200/csrc/ncc.cu /tmp/ncc_new.cu
for v in new old new old; do
  if [ $v = old ]; then cp tools/experiments/ab_old/ncc.cu paper_2009_04755_b200/csrc/ncc.cu; else cp /tmp/ncc_new.cu paper_2009_04755_b200/csrc/ncc.cu; fi
  python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
  timeout 600 python bench.py --app ncc --steps 5 --warmup 3 --no-cpu --no-e2e >> gpurun_out/r2x_ncc_$v.log 2>&1
done
tail -2 gpurun_out/r2x_tests.log
