# usage: bash tools/gpu_check.sh [tag]  — gpu tests, a bench line and a launch list
tag=${1:-x}
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py --no-cpu ${BENCH_ARGS} > gpurun_out/bench_$tag.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_$tag.log | cut -c1-1500
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python tools/prof_step.py --steps 3 --decode 256 --decode-mode tensor > /dev/null 2>&1; echo launches=$?
