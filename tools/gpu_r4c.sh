# MMA issuer warps on sub-partitions 2/3 (-DNVOL_M4_SKEW=2: two idle warps before them) vs 0/1
# (the skew knob was removed after this measurement: slightly slower)
export PYTHONUNBUFFERED=1
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_M4_SKEW=2 2>&1 | grep error
timeout 600 python -m pytest tests/test_gpu_tc_parity.py -q -x 2>&1 | tail -1
for ex in "" "-DNVOL_M4_SKEW=2" "" "-DNVOL_M4_SKEW=2" "" "-DNVOL_M4_SKEW=2"; do
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="$ex" 2>&1 | grep error
timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_sk.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_sk.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[$ex]', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'mlp' in a})"; done
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error; true
