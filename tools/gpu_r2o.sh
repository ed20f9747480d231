# A/B: split-fp16 vs plain fp16 training forward (NVOL_MLP_SPLIT), timeline + bench + tc parity
export PYTHONUNBUFFERED=1
tag=${1:-r2o}
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_TIMELINE 2>&1 | grep error
for sp in 1 0; do NVOL_MLP_SPLIT=$sp python tools/timeline_mlp4.py > gpurun_out/tl_split${sp}_$tag.txt 2>&1; head -2 gpurun_out/tl_split${sp}_$tag.txt; done
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error
for sp in 1 0; do NVOL_MLP_SPLIT=$sp timeout 300 python bench.py --steps 50 --no-decode --no-render --no-cfg5 --no-cpu --no-simt > gpurun_out/bench_split${sp}_$tag.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_split${sp}_$tag.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('split $sp', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), {a: round(b*1e3,1) for a,b in k.items()}, 'e2e', round(d['e2e']['value']/1e6,1))"; done
NVOL_MLP_SPLIT=0 timeout 900 python -m pytest tests/test_gpu_tc_parity.py -q -x -rs --timeout 800 -k "not ensemble" > gpurun_out/pytest_tc_split0_$tag.log 2>&1; echo tcpar=$?; tail -3 gpurun_out/pytest_tc_split0_$tag.log
NVOL_MLP_SPLIT=0 python tools/psnr_diag.py --seeds 12 --modes 1 > gpurun_out/psnr_diag_split0_$tag.log 2>&1; head -c 300 gpurun_out/psnr_diag_split0_$tag.log
