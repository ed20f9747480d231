export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/render_launches_warm.csv python tools/prof_render.py tensor 2>&1 | grep -v "^==PROF==" | tail -1
python tools/summ_launch.py gpurun_out/render_launches_warm.csv
python tools/launches.py gpurun_out/render_launches_warm.csv 2>/dev/null | head -34
timeout 900 ncu --profile-from-start off --set full --cache-control none --clock-control none --import-source on -k regex:"rm_coord" -s 1 -c 1 -o gpurun_out/prof_rm_coord python tools/prof_render.py tensor > /dev/null 2>&1; echo p=$?
