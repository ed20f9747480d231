# round-robin blocking MMA issuer (NVOL_MMA_RR) A/B: timeline, bench, parity
export PYTHONUNBUFFERED=1
tag=${1:-r3a}
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_TIMELINE 2>&1 | grep error
for rr in 1 0; do NVOL_MMA_RR=$rr python tools/timeline_mlp4.py > gpurun_out/tl_rr${rr}_$tag.txt 2>&1; head -1 gpurun_out/tl_rr${rr}_$tag.txt; done
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error
for rr in 1 0 1 0; do NVOL_MMA_RR=$rr timeout 300 python bench.py --steps 100 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_rr${rr}_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_rr${rr}_$tag.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('rr $rr', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), {a: round(b*1e3,1) for a,b in k.items() if 'mlp' in a})"; done
NVOL_MMA_RR=1 timeout 600 python -m pytest tests/test_gpu_tc_parity.py tests/test_gpu_parity.py -q -x --timeout 500 -k "not ensemble and not converges" > gpurun_out/pytest_$tag.log 2>&1; echo tcpar=$?; tail -1 gpurun_out/pytest_$tag.log
