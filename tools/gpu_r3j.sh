# A/B on one box: one vs two MMA-issuing warps (NVOL_MMA_WARPS)
export PYTHONUNBUFFERED=1
for w in 1 2 1 2 1 2; do NVOL_MMA_WARPS=$w timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_mw$w.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_mw$w.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('mma warps $w', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'mlp' in a}, 'e2e', round(d['e2e']['value']/1e6,1))"; done
NVOL_MMA_WARPS=1 timeout 600 python -m pytest tests/test_gpu_tc_parity.py -q -x --timeout 500 -k "not ensemble" > gpurun_out/pytest_mw1.log 2>&1; echo tcpar1=$?; tail -1 gpurun_out/pytest_mw1.log
