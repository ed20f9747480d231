export PYTHONUNBUFFERED=1
for v in 0 1; do
  touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_ACT_LO=$v 2>&1 | grep error
  echo "== NVOL_ACT_LO=$v"
  python -m pytest tests -m gpu -q -k "tcgen05 or host_feed or train" 2>&1 | tail -3
  python tools/diag_tc.py 2>&1 | tail -4
  python bench.py --no-cpu --no-decode --no-render --no-cfg5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms']['mlp_tc_kernel'])"
done
