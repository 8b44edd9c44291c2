# round-1 evidence for the packed-f32x2 kernel on one GPU: bench line, launch list,
# full ncu of one pce_cluster launch (each only after the plain command exited 0)
set -x
timeout 900 python bench.py > gpurun_out/f2_bench.log 2>&1; echo BENCH $? >> gpurun_out/f2_bench.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/f2_ncu_list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pce_cluster -s 6 -c 1 -o gpurun_out/prof_f2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/f2_ncu_full.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/f2_reference.log 2>&1
