# encoder item order: level-major (default) vs tile-major (-DNVOL_ENCODE_TILE_MAJOR): encode time
# (the experiment flag was removed after this measurement: DESIGN.md "Where the step stands")
export PYTHONUNBUFFERED=1
for ex in "" "-DNVOL_ENCODE_TILE_MAJOR" "" "-DNVOL_ENCODE_TILE_MAJOR"; do
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="$ex" 2>&1 | grep error
[ "$ex" = "-DNVOL_ENCODE_TILE_MAJOR" ] && timeout 300 python -m pytest tests/test_gpu_tc_parity.py -q -x -k "encoder" 2>&1 | tail -1
timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_enc.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_enc.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[$ex]', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'encode' in a})"; done
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error; true
