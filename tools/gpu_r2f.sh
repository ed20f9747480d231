export PYTHONUNBUFFERED=1
tag=${1:-r2f}
timeout 1200 python -m pytest tests -m gpu -q -rs --timeout 900 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo bench=$?; tail -c 300 gpurun_out/bench_$tag.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$tag.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1; echo launches=$?
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"mlp_tc4" -s 2 -c 1 -o gpurun_out/prof_mlp4_$tag python tools/prof_step.py --steps 3 > /dev/null 2>&1; echo prof=$?
