# 2 GPUs: multi-GPU tests, C2 scaling line, home-only PCE and NCC paths at reduced N
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/r2e_topo.txt 2>&1
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q > gpurun_out/r2e_mgpu_tests.log 2>&1; echo T $? >> gpurun_out/r2e_mgpu_tests.log
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2e_c2_2gpu.log 2>&1; echo B $? >> gpurun_out/r2e_c2_2gpu.log
timeout 900 python bench.py --gpus 2 --home-only --items 1024 --side 2048 --steps 1 --warmup 1 --no-cpu > gpurun_out/r2e_pce_home.log 2>&1; echo P $? >> gpurun_out/r2e_pce_home.log
timeout 900 python bench.py --gpus 2 --app ncc --home-only --items 2048 --side 2048 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2e_ncc_home.log 2>&1; echo N $? >> gpurun_out/r2e_ncc_home.log
timeout 900 python bench.py --gpus 2 --app ncc --steps 3 --warmup 3 --no-cpu > gpurun_out/r2e_ncc_c2.log 2>&1; echo N2 $? >> gpurun_out/r2e_ncc_c2.log
for f in r2e_mgpu_tests r2e_c2_2gpu r2e_pce_home r2e_ncc_home r2e_ncc_c2; do echo == $f; tail -c 600 gpurun_out/$f.log; done
