# A/B of the fused Adam + next-encode step tail (NVOL_FUSED_TAIL) and its Adam-CTA share
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "fused_adam_encode or train_step_api or host_feed or deterministic" > gpurun_out/fused_pytest.log 2>&1; tail -3 gpurun_out/fused_pytest.log
for cfg in "0 0.5" "1 0.5" "1 0.3" "1 0.7"; do
  set -- $cfg
  echo "== fused $1 adam_frac $2"
  NVOL_FUSED_TAIL=$1 NVOL_AE_ADAM_FRAC=$2 timeout 300 python bench.py --no-cpu --no-decode --no-render --no-cfg5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernel_ms']), d['e2e']['ms_per_step'])"
done
