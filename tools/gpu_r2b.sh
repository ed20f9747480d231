# MLP v4 bring-up: correctness first (short timeouts), then A/B timing of the stage kernels
export PYTHONUNBUFFERED=1
tag=${1:-r2b}
timeout 300 python -m pytest tests/test_gpu_tc_parity.py -q -x -rs --timeout 240 -k "not psnr" -s > gpurun_out/pytest_tc_$tag.log 2>&1; echo tc=$?; tail -3 gpurun_out/pytest_tc_$tag.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contracts.py -q -rs --timeout 500 > gpurun_out/pytest_par_$tag.log 2>&1; echo par=$?; tail -3 gpurun_out/pytest_par_$tag.log
for v in 1 0; do NVOL_MLP4=$v timeout 300 python bench.py --steps 50 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_mlp4_${v}_$tag.log 2>&1; echo bench$v=$?; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_mlp4_${v}_$tag.log').read().strip().splitlines()[-1]); print('mlp4=$v', d['value']/1e6, d['ms_per_step'], d['roofline']['kernel_ms'])"; done
