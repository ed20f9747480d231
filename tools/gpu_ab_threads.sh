export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_c.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_c.log
for v in 512 256; do
  touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_TC_THREADS=$v 2>&1 | grep error
  timeout 600 python bench.py --no-cpu --no-decode --no-render > gpurun_out/bench_c$v.log 2>&1; echo bench$v=$?; tail -1 gpurun_out/bench_c$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$v.csv python tools/prof_step.py --steps 3 > /dev/null 2>&1
done
