export PYTHONUNBUFFERED=1
tag=${1:-r2v}
for fa in 1 0 1 0; do NVOL_FORK_AFTER_ENCODE=$fa timeout 300 python bench.py --steps 100 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_fa${fa}_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_fa${fa}_$tag.log').read().strip().splitlines()[-1]); e=d['e2e']; print('fork-after-encode $fa', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), 'e2e', round(e['value']/1e6,1), round(e['ms_per_step']*1e3,1), 'loss', round(d['final_loss'],5))"; done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -k "not ensemble" > gpurun_out/pytest_$tag.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_$tag.log
