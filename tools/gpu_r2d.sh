export PYTHONUNBUFFERED=1
tag=${1:-r2d}
for v in 1 0; do NVOL_MLP4=$v timeout 300 python -m pytest tests/test_gpu_tc_parity.py -q -x -rs -s --timeout 240 -k "gradients" > gpurun_out/pytest_tc_${v}_$tag.log 2>&1; echo tc$v=$?; grep "'pred'" gpurun_out/pytest_tc_${v}_$tag.log | head -2; done
for v in 1 0; do NVOL_MLP4=$v timeout 300 python bench.py --steps 50 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_mlp4_${v}_$tag.log 2>&1; echo bench$v=$?; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_mlp4_${v}_$tag.log').read().strip().splitlines()[-1]); print('mlp4=$v', d['value']/1e6, d['ms_per_step'], d['roofline']['kernel_ms'])"; done
