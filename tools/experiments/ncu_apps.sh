# ncu --set full of the final GMM / CV / 2048^2 PCE kernels (one launch each)
set -x
ncu --set full --clock-control none -k regex:gmm_pair -s 5 -c 1 -o gpurun_out/prof_gmm2 python bench.py --app gmm --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_gmm2.log 2>&1
ncu --set full --clock-control none -k regex:cv_work -s 20 -c 1 -o gpurun_out/prof_cv2 python tools/gap_trace.py cv --runs 1 > gpurun_out/ncu_cv2.log 2>&1
ncu --set full --clock-control none -k regex:pce2k_pair -s 1 -c 1 -o gpurun_out/prof_pce2k python bench.py --items 300 --side 2048 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_pce2k.log 2>&1
