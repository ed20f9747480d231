# Adam: the sweep's last N MB of parameters stored evict_last (kept in L2 for the next encode)
# (the experiment flag was removed after this measurement: no effect)
export PYTHONUNBUFFERED=1
for ex in ${AB:-"" "-DNVOL_ADAM_P_KEEP_MB=8" "-DNVOL_ADAM_P_KEEP_MB=16" "-DNVOL_ADAM_P_KEEP_MB=32" ""}; do
touch paper_2207_11620_b200/csrc/mlp.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="$ex" 2>&1 | grep error
timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_pk.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_pk.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[$ex]', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'encode' in a or 'adam' in a})"; done
touch paper_2207_11620_b200/csrc/mlp.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error; true
