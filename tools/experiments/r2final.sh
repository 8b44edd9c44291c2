# final-code evidence: C2 bench line, ncu launch list of the C2 bench, ncu --set full of one job launch per PCE kernel
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2final_build.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2final_c2.log 2>&1
timeout 600 python bench.py --items 512 --side 2048 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2final_2k.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2final_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r2final_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pce_cluster -s 14 -c 1 -o gpurun_out/r2final_prof_pce python bench.py --items 1024 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2final_ncu_pce.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pce2k_pair -s 14 -c 1 -o gpurun_out/r2final_prof_pce2k python bench.py --items 512 --side 2048 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2final_ncu_pce2k.log 2>&1
ls -la gpurun_out/
