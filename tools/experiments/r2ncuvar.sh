# pce2k under ncu: per-launch time / DRAM / L2 hit for PCE2K_ROW_ARRIVE=0 vs 1 and with the round barrier off
set -x
cd $GRAFT_REPO_ROOT
B="import sys; sys.path.insert(0,'paper_2009_04755_b200'); import _build; _build.build(force=True)"
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
for v in 0 1; do
  RK_NVCC_FLAGS="-DPCE2K_ROW_ARRIVE=$v" python -c "$B"
  timeout 600 ncu --metrics $M --clock-control none -k regex:pce2k_pair -s 12 -c 4 --csv python bench.py --items 512 --side 2048 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2ncuvar_a$v.csv 2>&1
done
RK_PCE_LOCKSTEP=0 timeout 600 ncu --metrics $M --clock-control none -k regex:pce2k_pair -s 12 -c 4 --csv python bench.py --items 512 --side 2048 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > gpurun_out/r2ncuvar_nolock.csv 2>&1
