export PYTHONUNBUFFERED=1
for b in 1 4 6 8; do
  touch paper_2207_11620_b200/csrc/mlp.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_ADAM_MINB=$b 2>&1 | grep error
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_a$b.csv python tools/prof_step.py --steps 3 > /dev/null 2>&1
  echo "minb $b"; python tools/launches2.py gpurun_out/launches_a$b.csv 1
done
