#!/bin/bash
# Usage (under gpurun): tools/gpu_prof.sh <tag> <kernel-regex> [bench args...]
# Plain run first (must exit 0), then one ncu --set full capture of the matching kernels.
tag=$1; shift; kre=$1; shift; skip=${SKIP:-40}; cnt=${COUNT:-2}
args="$@"
python bench.py $args > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c $cnt \
    -o gpurun_out/prof_$tag python bench.py $args > gpurun_out/ncu_$tag.log 2>&1
echo "prof exit $?" >> gpurun_out/ncu_$tag.log
