set -x
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/r2t_tests.log 2>&1; echo TESTS $? >> gpurun_out/r2t_tests.log
tail -14 gpurun_out/r2t_tests.log
