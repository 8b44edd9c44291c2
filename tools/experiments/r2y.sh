# pce2k: radix-2 twiddles from a shared table (new) vs W^lane * W_64^k1 products (old); 2048^2 tests + A/B
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_pce_gpu.py -q -k "2048" > gpurun_out/r2y_tests.log 2>&1
timeout 300 python tools/pce_determinism.py --side 2048 --n 24 --runs 2 > gpurun_out/r2y_det.log 2>&1
cp paper_2009_04755_b200/csrc/pce2k.cu /tmp/n_pce2k.cu; cp paper_2009_04755_b200/csrc/fft.cuh /tmp/n_fft.cuh
for v in new old new old; do
  if [ $v = old ]; then cp tools/experiments/ab_old/pce2k.cu paper_2009_04755_b200/csrc/pce2k.cu; cp tools/experiments/ab_old/fft.cuh paper_2009_04755_b200/csrc/fft.cuh;
  else cp /tmp/n_pce2k.cu paper_2009_04755_b200/csrc/pce2k.cu; cp /tmp/n_fft.cuh paper_2009_04755_b200/csrc/fft.cuh; fi
  python -c "import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
  timeout 600 python bench.py --items 384 --side 2048 --steps 1 --warmup 2 --no-e2e --no-cpu --no-parity >> gpurun_out/r2y_2k_$v.log 2>&1
done
tail -2 gpurun_out/r2y_tests.log; cut -c 1-200 gpurun_out/r2y_det.log
