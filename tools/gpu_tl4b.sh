export PYTHONUNBUFFERED=1
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_TIMELINE 2>&1 | grep error
python tools/timeline_mlp4.py > gpurun_out/tl4b.txt 2>&1; head -3 gpurun_out/tl4b.txt
