# mbarrier try_wait suspend-time hint of the MLP's blocking waits: 1e6 ns (default), 1e4, 1e3, none
# (the hint knob was removed after this measurement: no effect)
export PYTHONUNBUFFERED=1
for ex in "" "-DNVOL_MBAR_HINT=10000" "-DNVOL_MBAR_HINT=1000" "-DNVOL_MBAR_NOHINT" ""; do
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="$ex" 2>&1 | grep error
timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_mb.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_mb.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[$ex]', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'mlp' in a})"; done
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error; true
