# 2048^2: does the pair order within a launch (leaf size) change DRAM traffic / time of pce2k_pair?
set -x
cd $GRAFT_REPO_ROOT
for leaf in 8 12 16; do
  timeout 600 python bench.py --items 384 --side 2048 --leaf $leaf --steps 1 --warmup 2 --no-e2e --no-cpu --no-parity > gpurun_out/r2j_bench_leaf$leaf.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pce2k_pair -s 6 -c 3 --csv python bench.py --items 384 --side 2048 --leaf $leaf --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2j_ncu_leaf$leaf.csv 2>&1
done
for leaf in 8 12 16; do grep -h '"value"' gpurun_out/r2j_bench_leaf$leaf.log | cut -c 1-120; grep -h "pce2k_pair" gpurun_out/r2j_ncu_leaf$leaf.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | head -12; done
