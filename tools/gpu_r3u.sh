# dW partials folded by the scatter prologue (default) vs REDs from the MLP kernel (NVOL_DW_PARTIALS=0):
# parity tests, then a same-box bench A/B
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tc_parity.py tests/test_gpu_contracts.py tests/test_gpu_dp.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for v in 1 0 1 0; do
NVOL_DW_PARTIALS=$v timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_dwp.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_dwp.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[DW_PARTIALS=$v]', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'mlp' in a or 'scatter' in a}, 'e2e', round(d['e2e']['value']/1e6,1))"; done
