export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_j.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu_j.log
for v in 1 0; do
  NVOL_SAMPLE_OVERLAP=$v timeout 600 python bench.py --no-cpu --no-decode --no-render > gpurun_out/bench_j$v.log 2>&1; echo bench$v=$?; tail -1 gpurun_out/bench_j$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['final_loss'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_j.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1
