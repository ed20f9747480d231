export PYTHONUNBUFFERED=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_h.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1; echo l=$?
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"scatter_kernel" -s 2 -c 1 -o gpurun_out/prof_scatter_h python tools/prof_step.py --steps 4 > /dev/null 2>&1; echo p=$?
