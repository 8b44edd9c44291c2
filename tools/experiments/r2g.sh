# 1 GPU: tests, headline bench, reference arm, app lines, ncu launch list + full capture of pce_cluster
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2g_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2g_tests.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2g_bench.log 2>&1; echo BENCH $? >> gpurun_out/r2g_bench.log
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r2g_ref.log 2>&1
timeout 900 python bench.py --app gmm --steps 5 --warmup 3 > gpurun_out/r2g_gmm.log 2>&1
timeout 900 python bench.py --app cv --steps 3 --warmup 3 > gpurun_out/r2g_cv.log 2>&1
timeout 600 python bench.py --impl reference --app gmm --steps 5 --warmup 3 > gpurun_out/r2g_ref_gmm.log 2>&1
timeout 600 python bench.py --impl reference --app cv --steps 5 --warmup 3 > gpurun_out/r2g_ref_cv.log 2>&1
timeout 600 python bench.py --impl reference --items 128 --side 256 --steps 5 --warmup 3 > gpurun_out/r2g_ref_c1.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2g_ncu_list.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:pce_cluster -s 6 -c 1 -o gpurun_out/r2g_pce python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2g_ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pce2k_pair -s 2 -c 1 -o gpurun_out/r2g_pce2k python bench.py --items 256 --side 2048 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2g_ncu_2k.log 2>&1
ls -la gpurun_out/ | tail -20
