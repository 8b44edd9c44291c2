# leaf size A/B at 2048^2 (same box, N = 512), two rounds
for r in 1 2; do for lf in 8 12 16 4; do
  timeout 600 python bench.py --items 512 --side 2048 --leaf $lf --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/leaf2k_$lf.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/leaf2k_$lf.log').read().strip().splitlines()[-1]); print('leaf $lf', round(d['value']), d['roofline']['ms_per_launch'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" | tee -a gpurun_out/leaf2k_summary.log
done; done
