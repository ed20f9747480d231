# split-fp16 vs plain fp16 training forward with two MMA issuers (same box), parity bars
export PYTHONUNBUFFERED=1
for sp in 1 0 1 0; do NVOL_MLP_SPLIT=$sp timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_sp$sp.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_sp$sp.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('split $sp', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'mlp' in a})"; done
NVOL_MLP_SPLIT=0 timeout 900 python -m pytest tests/test_gpu_tc_parity.py -q -rs -s --timeout 800 -k "not ensemble" > gpurun_out/pytest_sp0.log 2>&1; echo tcpar=$?; grep "passed\|failed" gpurun_out/pytest_sp0.log | tail -2; grep -o "{'pred'.*" gpurun_out/pytest_sp0.log | head -2 | cut -c1-400
