export PYTHONUNBUFFERED=1
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="-DNVOL_TIMELINE -DNVOL_TIMELINE_CLOCK" 2>&1 | grep error
python tools/timeline_mlp4.py > gpurun_out/tl_clock.txt 2>&1; head -24 gpurun_out/tl_clock.txt; grep "slot 0 epi" gpurun_out/tl_clock.txt | head -8
