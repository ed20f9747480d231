export PYTHONUNBUFFERED=1
tag=${1:-r2}
timeout 2400 python tools/run_reference_tests.py --run $tag > gpurun_out/reftests_$tag.log 2>&1; echo reftests=$?; tail -3 gpurun_out/reftests_$tag.log
