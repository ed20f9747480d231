export PYTHONUNBUFFERED=1
for v in 0 1 2 3 0 1; do
  touch paper_2207_11620_b200/csrc/mlp.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_ADAM_L2=$v 2>&1 | grep error
  echo "== NVOL_ADAM_L2=$v"
  python bench.py --no-cpu --no-decode --no-render --steps 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_p1.csv python tools/prof_step.py --steps 3 > /dev/null 2>&1
python tools/launches2.py gpurun_out/launches_p1.csv 5
