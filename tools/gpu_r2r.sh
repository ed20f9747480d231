# PDL A/B (NVOL_PDL) + the GPU suite with PDL on
export PYTHONUNBUFFERED=1
tag=${1:-r2r}
for pd in 1 0 1 0; do NVOL_PDL=$pd timeout 300 python bench.py --steps 100 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_pdl${pd}_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_pdl${pd}_$tag.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('pdl $pd', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), {a: round(b*1e3,1) for a,b in k.items()}, 'e2e', round(d['e2e']['value']/1e6,1))"; done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "not ensemble" > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_$tag.log
