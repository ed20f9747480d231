export PYTHONUNBUFFERED=1
for v in old new; do
  cp /tmp/infer_$v.cu paper_2207_11620_b200/csrc/infer_tc.cu   # A/B sources staged under /tmp by the caller
  make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error
  echo "== $v"; timeout 300 python tools/decode_time.py 2>&1 | tail -1
done
