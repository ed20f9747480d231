# usage: bash tools/gpu_prof_k.sh <kernel-regex> <tag> [skip]  — one ncu --set full capture of a training kernel
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${3:-1} -c 1 \
    -o gpurun_out/prof_$2 python tools/prof_step.py --steps 3 > gpurun_out/prof_$2.log 2>&1; echo prof=$?
