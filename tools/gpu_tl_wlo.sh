export PYTHONUNBUFFERED=1
for w in 1 0; do
  touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="-DNVOL_TIMELINE -DNVOL_FWD_WLO=$w" 2>&1 | grep error
  echo "== WLO=$w"; python tools/timeline_mlp.py > gpurun_out/tl_$w.txt 2>&1; head -1 gpurun_out/tl_$w.txt; grep "mma 1[0-9] \|epi 16" gpurun_out/tl_$w.txt | head -4
  touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="-DNVOL_FWD_WLO=$w" 2>&1 | grep error
  timeout 600 python -m pytest tests -m gpu -x -q -k "tcgen05 or tensor" 2>&1 | tail -2
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f$w.csv python tools/prof_step.py --steps 2 > /dev/null 2>&1
  python tools/launches.py gpurun_out/launches_f$w.csv | grep nvol | tail -6
done
