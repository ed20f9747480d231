export PYTHONUNBUFFERED=1
tag=${1:-r2h}
timeout 900 python -m pytest tests -m gpu -q -rs --timeout 600 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_$tag.log
for r in "8 2" "1 2" "4 2" "8 3" "16 2"; do set -- $r; NVOL_SC_REP=$1 NVOL_SC_REP_LEVELS=$2 timeout 300 python bench.py --steps 50 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_rep_$1_$2_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_rep_$1_$2_$tag.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('rep $1 lv $2', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), 'scatter', round(k['scatter_kernel']*1e3,1), 'mlp', round(k['mlp_tc_kernel']*1e3,1), 'e2e', round(d['e2e']['value']/1e6,1))"; done
