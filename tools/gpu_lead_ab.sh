export PYTHONUNBUFFERED=1
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 2 0 2 0; do
  echo "== lead $v"
  NVOL_FLAT_LEAD=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_l$v.csv python tools/prof_step.py --steps 3 > /dev/null 2>&1
  python tools/launches2.py gpurun_out/launches_l$v.csv 4
  NVOL_FLAT_LEAD=$v python bench.py --no-cpu --no-decode --no-render 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
