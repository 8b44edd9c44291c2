# leaf size A/B on the current kernel (same box, C2 subset N = 2,048), two rounds
for r in 1 2; do for lf in 8 12 16 24; do
  timeout 600 python bench.py --items 2048 --leaf $lf --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/leaf2_$lf.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/leaf2_$lf.log').read().strip().splitlines()[-1]); print('leaf $lf', round(d['value']), d['roofline']['ms_per_launch'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" | tee -a gpurun_out/leaf2_summary.log
done; done
