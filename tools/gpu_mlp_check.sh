export PYTHONUNBUFFERED=1
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu --no-decode --no-render 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_m.csv python tools/prof_step.py --steps 3 > /dev/null 2>&1
python tools/launches2.py gpurun_out/launches_m.csv 5
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_TIMELINE 2>&1 | grep error; python tools/timeline_mlp.py > gpurun_out/tl_m.txt 2>&1; head -1 gpurun_out/tl_m.txt
