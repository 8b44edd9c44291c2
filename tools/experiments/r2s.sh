# PCE launch order grouped by the left item (RK_PAIR_ORDER=1) vs leaf order (0): 1024^2 and 2048^2, plus DRAM bytes
set -x
cd $GRAFT_REPO_ROOT
for v in 1 0 1 0; do
  RK_PAIR_ORDER=$v timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-parity >> gpurun_out/r2s_c2_o$v.log 2>&1
  RK_PAIR_ORDER=$v timeout 600 python bench.py --items 384 --side 2048 --steps 1 --warmup 2 --no-e2e --no-cpu --no-parity >> gpurun_out/r2s_2k_o$v.log 2>&1
done
for v in 1 0; do
  RK_PAIR_ORDER=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pce2k_pair -s 6 -c 2 --csv python bench.py --items 384 --side 2048 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2s_ncu2k_o$v.csv 2>&1
  RK_PAIR_ORDER=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pce_cluster -s 20 -c 2 --csv python bench.py --items 1024 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2s_ncu1k_o$v.csv 2>&1
done
for f in c2 2k; do for v in 1 0; do python -c "
import json
for l in open('gpurun_out/r2s_${f}_o$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$f o$v', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], round(d['value']/d['clocks']['sm_mhz'],2))"; done; done
