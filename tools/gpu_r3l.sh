# flakiness check of the statistical GPU tests (5 repetitions)
export PYTHONUNBUFFERED=1
for i in 1 2 3 4 5; do timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_parity.py -q -s --timeout 800 -k "converges or ensemble or psnr" 2>&1 | grep -E "passed|failed|gpu_mean|Error" | cut -c1-300; done
