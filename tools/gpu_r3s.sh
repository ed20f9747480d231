# Adam vs optimizer-state layout (timing experiment, tools/adam_layout.py)
export PYTHONUNBUFFERED=1
for l in 0 1 2 0; do
touch paper_2207_11620_b200/csrc/mlp.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="$([ $l = 0 ] || echo -DNVOL_ADAM_LAYOUT_EXPT=$l)" 2>&1 | grep error
timeout 300 python tools/adam_layout.py $l 2>&1 | tail -1
done
touch paper_2207_11620_b200/csrc/mlp.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error
