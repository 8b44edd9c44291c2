# 4-GPU box: multi-GPU parity tests, then the C2 bench at N=4 and N=2 (round-1 final-build check)
mkdir -p gpurun_out
python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/mg_tests.log 2>&1; echo mgtests=$?; tail -2 gpurun_out/mg_tests.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 > gpurun_out/bench4_final.json 2> gpurun_out/bench4_final.err; echo b4=$?; tail -1 gpurun_out/bench4_final.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 > gpurun_out/bench2_final.json 2> gpurun_out/bench2_final.err; echo b2=$?; tail -1 gpurun_out/bench2_final.json
