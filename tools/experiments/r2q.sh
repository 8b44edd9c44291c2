# 2 GPUs: P2P mechanisms with NVLink counters; ncu of the NCC Gram, CV merge and GMM kernels (one GPU)
set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/p2p_bw.py > gpurun_out/r2q_p2p.log 2>&1
export CUDA_VISIBLE_DEVICES=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ncc_gram2 -s 40 -c 1 -o gpurun_out/r2q_ncc python bench.py --app ncc --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2q_ncu_ncc.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:cv_work -s 4 -c 1 -o gpurun_out/r2q_cv python bench.py --app cv --items 600 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2q_ncu_cv.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:gmm_pair -s 20 -c 1 -o gpurun_out/r2q_gmm python bench.py --app gmm --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2q_ncu_gmm.log 2>&1
tail -2 gpurun_out/r2q_p2p.log | cut -c 1-1500; ls gpurun_out/r2q*
