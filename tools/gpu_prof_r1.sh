# ncu evidence for round 1: launch list + one --set full capture per hot kernel
set -x
export PYTHONUNBUFFERED=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv \
    python tools/prof_step.py --steps 3 --decode 256 --decode-mode tensor > gpurun_out/launches_r1.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on \
    -k regex:"adam_flat|scatter_kernel|mlp_tc_kernel|encode_tiles|sample_incore|reduce_partials" -s 9 -c 9 \
    -o gpurun_out/prof_step_r1 python tools/prof_step.py --steps 3 > gpurun_out/prof_step_r1.log 2>&1; echo full=$?
ncu --set full --clock-control none --import-source on -k regex:"infer_tc_kernel" -s 2 -c 1 \
    -o gpurun_out/prof_decode_r1 python tools/prof_step.py --steps 1 --decode 256 --decode-mode tensor > gpurun_out/prof_decode_r1.log 2>&1; echo dec=$?
ls -la gpurun_out
