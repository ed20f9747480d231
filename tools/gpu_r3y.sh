# copies of the MLP weight image in global memory: 8 (default) vs 1 (NVOL_IMG_COPIES)
# (the copies knob was removed after this measurement: no change in the step)
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tc_parity.py tests/test_gpu_contracts.py -q -x 2>&1 | tail -1
for v in 8 1 8 1; do
NVOL_IMG_COPIES=$v timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_img.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_img.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[copies $v]', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'mlp' in a}, 'e2e', round(d['e2e']['value']/1e6,1))"; done
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_TIMELINE 2>&1 | grep error; python tools/timeline_mlp4.py 2>&1 | head -1; NVOL_IMG_COPIES=1 python tools/timeline_mlp4.py 2>&1 | head -1
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error; true
