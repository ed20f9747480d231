export PYTHONUNBUFFERED=1
for v in 0 1; do
  touch paper_2207_11620_b200/csrc/mlp.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_ADAM_UNROLL2=$v 2>&1 | grep error
  timeout 600 python bench.py --no-cpu --no-decode --no-render > gpurun_out/bench_k$v.log 2>&1; echo bench$v=$?; tail -1 gpurun_out/bench_k$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_k$v.csv python tools/prof_step.py --steps 3 > /dev/null 2>&1
  python tools/launches2.py gpurun_out/launches_k$v.csv 5
done
