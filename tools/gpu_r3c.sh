export PYTHONUNBUFFERED=1
tag=${1:-r3c}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu_$tag.log
timeout 2400 python tools/run_reference_tests.py --run $tag > gpurun_out/reftests_$tag.log 2>&1; echo reftests=$?; tail -2 gpurun_out/reftests_$tag.log
