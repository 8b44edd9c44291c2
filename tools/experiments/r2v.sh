# 4 GPUs: app lines (C4 GMM, C5 CV) and NCC C2 with the round-2 kernels
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --gpus 4 --app gmm --steps 5 --warmup 3 --no-cpu > gpurun_out/r2v_gmm4.log 2>&1
timeout 1200 python bench.py --gpus 4 --app cv --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2v_cv4.log 2>&1
timeout 900 python bench.py --gpus 4 --app ncc --steps 3 --warmup 3 --no-cpu > gpurun_out/r2v_ncc4.log 2>&1
timeout 900 python bench.py --gpus 2 --app gmm --steps 5 --warmup 3 --no-cpu > gpurun_out/r2v_gmm2.log 2>&1
for f in gmm4 cv4 ncc4 gmm2; do tail -c 300 gpurun_out/r2v_$f.log; echo; done
