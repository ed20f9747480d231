export PYTHONUNBUFFERED=1
tag=${1:-r2m}
python tools/traj_cfg2.py --steps 300 > gpurun_out/traj_$tag.log 2>&1; echo traj=$?
timeout 900 python -m pytest tests/test_gpu_cfg34.py -q -rs > gpurun_out/pytest_cfg34_$tag.log 2>&1; echo cfg34=$?; tail -3 gpurun_out/pytest_cfg34_$tag.log
timeout 2400 python tools/run_reference_tests.py --run $tag > gpurun_out/reftests_$tag.log 2>&1; echo reftests=$?; tail -3 gpurun_out/reftests_$tag.log
