export PYTHONUNBUFFERED=1
tag=${1:-r2g}
timeout 900 python -m pytest tests -m gpu -q -x -rs --timeout 600 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_$tag.log
for v in 1 0; do NVOL_MLP4=$v timeout 300 python bench.py --steps 50 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_mlp4_${v}_$tag.log 2>&1; echo bench$v=$?; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_mlp4_${v}_$tag.log').read().strip().splitlines()[-1]); print('mlp4=$v', d['value']/1e6, d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['value']/1e6)"; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$tag.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1; echo launches=$?; python tools/launches2.py gpurun_out/launches_$tag.csv 6 | tail -7
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_TIMELINE 2>&1 | grep error
python tools/timeline_mlp4.py > gpurun_out/tl4_$tag.txt 2>&1; head -2 gpurun_out/tl4_$tag.txt
