# fused encoder in the MLP kernel (NVOL_FUSED_ENC=1): parity + timeline + bench A/B
export PYTHONUNBUFFERED=1
tag=${1:-r2t}
NVOL_FUSED_ENC=1 timeout 600 python -m pytest tests/test_gpu_tc_parity.py -q -x -rs --timeout 500 -k "not ensemble" > gpurun_out/pytest_tc_$tag.log 2>&1; echo tcpar=$?; tail -2 gpurun_out/pytest_tc_$tag.log
for fe in 1 0 1; do NVOL_FUSED_ENC=$fe timeout 300 python bench.py --steps 100 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_fe${fe}_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_fe${fe}_$tag.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('fused $fe', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), {a: round(b*1e3,1) for a,b in k.items()}, 'e2e', round(d['e2e']['value']/1e6,1), 'loss', d['final_loss'])"; done
NVOL_FUSED_ENC=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_fe_$tag.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1; python tools/launches2.py gpurun_out/launches_fe_$tag.csv 6
