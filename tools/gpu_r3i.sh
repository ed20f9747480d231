# two MMA-issuing warps with round-robin suspended waits: timeline (clock), bench, tc parity
export PYTHONUNBUFFERED=1
tag=${1:-r3i}
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="-DNVOL_TIMELINE -DNVOL_TIMELINE_CLOCK" 2>&1 | grep error
python tools/timeline_mlp4.py > gpurun_out/tl_$tag.txt 2>&1; head -1 gpurun_out/tl_$tag.txt
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error
for i in 1 2; do timeout 300 python bench.py --steps 100 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$tag.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('bench', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), {a: round(b*1e3,1) for a,b in k.items() if 'mlp' in a})"; done
timeout 600 python -m pytest tests/test_gpu_tc_parity.py tests/test_gpu_parity.py -q -x --timeout 500 -k "not ensemble" > gpurun_out/pytest_$tag.log 2>&1; echo tcpar=$?; tail -1 gpurun_out/pytest_$tag.log
