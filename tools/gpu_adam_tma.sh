export PYTHONUNBUFFERED=1
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 1 0; do
  echo "== NVOL_ADAM_TMA=$v"
  NVOL_ADAM_TMA=$v python bench.py --no-cpu --no-decode --no-render 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms']['adam_step_kernel'], d['e2e']['value'], d['final_loss'])"
  NVOL_ADAM_TMA=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_t$v.csv python tools/prof_step.py --steps 3 > /dev/null 2>&1
  python tools/launches2.py gpurun_out/launches_t$v.csv 5
done
