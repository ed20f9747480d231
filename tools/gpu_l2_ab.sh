# step A/B: bench twice + warm launch list with DRAM bytes (scatter / encode L2 residency)
export PYTHONUNBUFFERED=1
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-decode --no-render --no-cfg5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernel_ms']))"; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --cache-control none --csv --log-file gpurun_out/launches_l2.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1
python tools/launches2.py gpurun_out/launches_l2.csv 5 2>/dev/null | tail -6
