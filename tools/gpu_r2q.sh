# A/B: Adam TMA ring geometry (NVOL_ADAM_CFG), bench step + Adam kernel time, Adam parity per config
export PYTHONUNBUFFERED=1
tag=${1:-r2q}
for c in 0 1 2 3 4 5; do NVOL_ADAM_CFG=$c timeout 300 python bench.py --steps 50 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_adam${c}_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_adam${c}_$tag.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('cfg $c', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), {a: round(b*1e3,1) for a,b in k.items()})"; done
for c in 1 2 3 4 5; do NVOL_ADAM_CFG=$c timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py -q -x -k "adam or nan" > gpurun_out/pytest_adam${c}_$tag.log 2>&1; echo adam$c=$? $(tail -1 gpurun_out/pytest_adam${c}_$tag.log); done
for c in 0 2 3; do NVOL_ADAM_CFG=$c timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_adam${c}_$tag.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1; python tools/launches2.py gpurun_out/launches_adam${c}_$tag.csv 12 | grep adam; done
