# 4 GPUs: P2P mechanisms, multi-GPU tests at world 4, C2 line, C3-Gram (NCC) and C3 PCE through bench.py
set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/p2p_bw.py > gpurun_out/r2f_p2p.log 2>&1
tail -2 gpurun_out/r2f_p2p.log
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q > gpurun_out/r2f_mgpu_tests.log 2>&1; echo T $? >> gpurun_out/r2f_mgpu_tests.log
timeout 900 python bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2f_c2_4gpu.log 2>&1; echo B $? >> gpurun_out/r2f_c2_4gpu.log
timeout 900 python bench.py --gpus 4 --app ncc --items 16384 --side 2048 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2f_c3ncc_ce.log 2>&1; echo N $? >> gpurun_out/r2f_c3ncc_ce.log
RK_PEER_COPY_CTAS=32 timeout 900 python bench.py --gpus 4 --app ncc --items 16384 --side 2048 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2f_c3ncc_k32.log 2>&1; echo N $? >> gpurun_out/r2f_c3ncc_k32.log
timeout 2400 python bench.py --gpus 4 --items 16384 --side 2048 --steps 1 --warmup 1 --no-cpu > gpurun_out/r2f_c3pce.log 2>&1; echo P $? >> gpurun_out/r2f_c3pce.log
for f in r2f_mgpu_tests r2f_c2_4gpu r2f_c3ncc_ce r2f_c3ncc_k32 r2f_c3pce; do echo == $f; tail -c 400 gpurun_out/$f.log; done
