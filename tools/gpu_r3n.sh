# scatter || Adam overlap micro-experiment at several scatter CTA sizes (register footprint)
export PYTHONUNBUFFERED=1
for t in 1024 768 512; do
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="-DNVOL_SC_THREADS=$t" 2>&1 | grep error
echo "SC_THREADS=$t"; timeout 300 python tools/overlap_sa.py 2>&1 | tail -2
done
