# Round evidence: gpu tests, full bench line, warm launch list, ncu --set full of the step kernels + decode
# usage: bash tools/gpu_round_evidence.sh <tag>
tag=${1:-r1}
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu_$tag.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$tag.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1; echo launches=$?
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"adam_tma|adam_step|mlp_tc|scatter_kernel|encode_tiles|sample_incore|pack_w4|dw_reduce" -s 7 -c 7 -o gpurun_out/prof_step_$tag python tools/prof_step.py --steps 3 > /dev/null 2>&1; echo prof=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:infer_tc_kernel -s 0 -c 1 -o gpurun_out/prof_decode_$tag python tools/prof_step.py --steps 1 --decode 256 --decode-mode tensor > /dev/null 2>&1; echo profd=$?
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/render_launches_$tag.csv python tools/prof_render.py tensor > /dev/null 2>&1; echo render_launches=$?
timeout 900 ncu --profile-from-start off --set full --cache-control none --clock-control none --import-source on -k regex:"rm_step|infer_tc" -s 0 -c 2 -o gpurun_out/prof_render_$tag python tools/prof_render.py tensor > /dev/null 2>&1; echo prof_render=$?
