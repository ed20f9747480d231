export PYTHONUNBUFFERED=1
for c in 3 2 1 0; do
  echo "== NVOL_SC_COARSE=$c"
  NVOL_SC_COARSE=$c timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c$c.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1
  python tools/launches.py gpurun_out/launches_c$c.csv | grep -E "scatter_kernel" | tail -2
done
