set -x
timeout 300 python tools/apps_bench.py gmm > gpurun_out/abg_tool.log 2>&1
timeout 300 python bench.py --app gmm --no-e2e --no-cpu > gpurun_out/abg_bench.log 2>&1
RK_NO_CLOCKS=1 timeout 300 python bench.py --app gmm --no-e2e --no-cpu > gpurun_out/abg_bench_noclk.log 2>&1
timeout 300 python tools/apps_bench.py gmm > gpurun_out/abg_tool2.log 2>&1
