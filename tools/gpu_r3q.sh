# Adam ring sweep at 3 CTAs/SM (chunk floats x stages), same box: in-step Adam and step time
export PYTHONUNBUFFERED=1
for ex in "" "-DNVOL_AD_CH=1024 -DNVOL_AD_ST=4" "-DNVOL_AD_CH=2048 -DNVOL_AD_ST=2" "-DNVOL_AD_CH=1536 -DNVOL_AD_ST=3" "" "-DNVOL_AD_CH=1024 -DNVOL_AD_ST=5"; do
touch paper_2207_11620_b200/csrc/mlp.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="$ex" 2>&1 | grep error
timeout 300 python bench.py --steps 200 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_ad.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_ad.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[$ex]', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), {a: round(b*1e3,1) for a,b in k.items() if 'adam' in a})"; done
