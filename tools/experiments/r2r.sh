# ncu of the NCC Gram kernel (CTA-pair tcgen05)
set -x
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gram -c 2 -o gpurun_out/r2r_ncc python tools/ncc_bench.py 4096 1024 > gpurun_out/r2r_ncu_ncc.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv python tools/ncc_bench.py 1024 1024 > gpurun_out/r2r_ncc_list.csv 2>&1
tail -5 gpurun_out/r2r_ncu_ncc.log; grep -c gram gpurun_out/r2r_ncc_list.csv
