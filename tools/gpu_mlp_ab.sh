# MLP kernel A/B: timeline span of CTA 0 + bench step time (+ tcgen05 parity tests)
export PYTHONUNBUFFERED=1
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="-DNVOL_TIMELINE" 2>&1 | grep error
python tools/timeline_mlp.py 2>&1 | head -1
touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc 2>&1 | grep error
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "tcgen05 or fused or trajectory" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-decode --no-render --no-cfg5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernel_ms']))"; done
