# Stride padding A/B: NCC Gram (slot stride) and PCE (slot + T strides), same box
set -x
for pad in 0 256 4096 65792; do
  RK_SLOT_PAD=$pad timeout 300 python tools/ncc_bench.py 4096 1024 > gpurun_out/pad_ncc_$pad.log 2>&1
done
for pad in 0 4096 65792; do
  RK_SLOT_PAD=$pad RK_T_PAD=$pad timeout 600 python bench.py --items 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/pad_pce_$pad.log 2>&1
done
RK_SLOT_PAD=0 RK_T_PAD=4096 timeout 600 python bench.py --items 2048 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/pad_pce_t4096.log 2>&1
