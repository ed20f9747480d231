# timing bound: the scatter's coarse-level flush (148 CTAs REDing into the same 46 KB) skipped
# (the experiment flag was removed after this measurement: DESIGN.md "Weight-gradient flush")
export PYTHONUNBUFFERED=1
for ex in "" "-DNVOL_SC_NOFLUSH_EXPT" "" "-DNVOL_SC_NOFLUSH_EXPT"; do
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="$ex" 2>&1 | grep error
timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_sc.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_sc.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[$ex]', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'scatter' in a})"; done
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error; true
