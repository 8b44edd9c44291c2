set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_peer_tier_gpu.py -q -k "home_chunks" > gpurun_out/r2hc.log 2>&1; tail -n 15 gpurun_out/r2hc.log
