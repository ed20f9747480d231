export PYTHONUNBUFFERED=1
tag=${1:-r2e}
timeout 300 python -m pytest tests/test_gpu_tc_parity.py -q -x -rs -s --timeout 240 -k "not psnr" > gpurun_out/pytest_tc_$tag.log 2>&1; echo tc=$?; grep "'pred'" gpurun_out/pytest_tc_$tag.log | cut -c1-300; tail -1 gpurun_out/pytest_tc_$tag.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rs --timeout 500 -k "tcgen05 or psnr or train" > gpurun_out/pytest_par_$tag.log 2>&1; echo par=$?; tail -2 gpurun_out/pytest_par_$tag.log
for v in 1 0; do NVOL_MLP4=$v timeout 300 python bench.py --steps 50 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_mlp4_${v}_$tag.log 2>&1; echo bench$v=$?; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_mlp4_${v}_$tag.log').read().strip().splitlines()[-1]); print('mlp4=$v', d['value']/1e6, d['ms_per_step'], d['roofline']['kernel_ms'])"; done
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_TIMELINE 2>&1 | grep error
python tools/timeline_mlp4.py > gpurun_out/tl4_$tag.txt 2>&1; head -1 gpurun_out/tl4_$tag.txt
