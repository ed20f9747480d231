export PYTHONUNBUFFERED=1
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_TIMELINE 2>&1 | grep error
for sl in 1 2; do for sp in 1 0; do NVOL_MLP_SLOTS=$sl NVOL_MLP_SPLIT=$sp python tools/timeline_mlp4.py > gpurun_out/tl_s${sl}_split${sp}.txt 2>&1; head -1 gpurun_out/tl_s${sl}_split${sp}.txt; done; done
