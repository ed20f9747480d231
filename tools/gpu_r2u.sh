export PYTHONUNBUFFERED=1
tag=${1:-r2u}
for i in 1 2; do timeout 300 python bench.py --steps 100 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$tag.log').read().strip().splitlines()[-1]); e=d['e2e']; print('bench', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), 'e2e', round(e['value']/1e6,1), round(e['ms_per_step']*1e3,1), 'api', round(e['train_step_api']['value']/1e6,1))"; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py tests/test_gpu_estimator.py tests/test_gpu_outofcore.py -q -x > gpurun_out/pytest_$tag.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_$tag.log
python tools/e2e_probe.py 2>&1 | head -3
