# A/B: Adam keeps params L2-resident (evict_last) or streams them
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_g.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu_g.log
for v in 0 1; do
  touch paper_2207_11620_b200/csrc/mlp.cu; make -s -C paper_2207_11620_b200/csrc EXTRA=-DNVOL_ADAM_P_KEEP=$v 2>&1 | grep error
  timeout 600 python bench.py --no-cpu --no-decode --no-render > gpurun_out/bench_g$v.log 2>&1; echo bench$v=$?; tail -1 gpurun_out/bench_g$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
done
