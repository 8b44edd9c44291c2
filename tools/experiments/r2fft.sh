set -x
cd $GRAFT_REPO_ROOT
./tools/fft_bench > gpurun_out/r2fft.log 2>&1; cat gpurun_out/r2fft.log
