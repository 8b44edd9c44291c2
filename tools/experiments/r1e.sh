set -x
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r1e_pytest.log 2>&1; echo PYTEST $? >> gpurun_out/r1e_pytest.log
timeout 900 python bench.py > gpurun_out/r1e_bench.log 2>&1; echo BENCH $? >> gpurun_out/r1e_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1e_ref.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1e_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r1e_ncu.log 2>&1
