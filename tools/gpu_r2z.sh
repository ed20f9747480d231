export PYTHONUNBUFFERED=1
tag=${1:-r2z}
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -k "not ensemble" > gpurun_out/pytest_$tag.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_$tag.log
timeout 300 python bench.py --steps 50 --no-decode --no-render --no-cfg5 --no-cpu > gpurun_out/bench_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$tag.log').read().strip().splitlines()[-1]); print('bench', round(d['value']/1e6,1), 'simt', d['simt_engine'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_simt_$tag.csv python tools/prof_step.py --mode 0 --steps 3 > /dev/null 2>&1
python tools/launches2.py gpurun_out/launches_simt_$tag.csv 60 | tail -34
