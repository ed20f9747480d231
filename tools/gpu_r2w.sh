export PYTHONUNBUFFERED=1
tag=${1:-r2w}
for cfg in "NVOL_ADAM_THREADS=256" "NVOL_ADAM_THREADS=512" "NVOL_ADAM_THREADS=128" "NVOL_ADAM_TMA=0" "NVOL_ADAM_THREADS=512" "NVOL_ADAM_THREADS=256"; do env $cfg timeout 300 python bench.py --steps 100 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$tag.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('$cfg', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), {a: round(b*1e3,1) for a,b in k.items() if 'adam' in a})"; done
NVOL_ADAM_THREADS=512 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py -q -x -k "adam or nan" > gpurun_out/pytest_$tag.log 2>&1; echo adam512=$? $(tail -1 gpurun_out/pytest_$tag.log)
