# in-shader tcgen05 marcher: render tests (bitwise vs tensor wavefront), cfg4 parity, bench render
export PYTHONUNBUFFERED=1
tag=${1:-r2x}
timeout 600 python -m pytest tests/test_gpu_render.py tests/test_gpu_cfg34.py tests/test_gpu_parity.py -q -x -rs -s -k "render or shader or cfg4 or cfg3 or tensor or decode or eval" > gpurun_out/pytest_$tag.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_$tag.log; grep "'arch'" gpurun_out/pytest_$tag.log
timeout 600 python bench.py --steps 20 --no-decode --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$tag.log').read().strip().splitlines()[-1]); r=d['render']; print({k: (round(v['frame_ms'],3), v['evals']) for k,v in r.items() if isinstance(v, dict)})"
