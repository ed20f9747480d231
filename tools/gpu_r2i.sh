export PYTHONUNBUFFERED=1
tag=${1:-r2i}
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py -q -rs --timeout 500 -k "adam or nan or train" > gpurun_out/pytest_adam_$tag.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_adam_$tag.log
for v in 1 0; do NVOL_ADAM_TMA=$v timeout 300 python bench.py --steps 50 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_tma_${v}_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_tma_${v}_$tag.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('tma $v', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), 'adam', round(k['adam_step_kernel']*1e3,1), 'scatter', round(k['scatter_kernel']*1e3,1), 'e2e', round(d['e2e']['value']/1e6,1), d['roofline']['frac'])"; done
NVOL_ADAM_TMA=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$tag.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1; echo launches=$?; python tools/launches2.py gpurun_out/launches_$tag.csv 6 | tail -7
