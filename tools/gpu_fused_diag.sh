export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python tools/stage_poll.py odd 8192 L1 2>&1 | tail -2
timeout 400 python -m pytest tests/test_gpu_parity.py -x -v -k "fused_adam_encode or tcgen05_step" > gpurun_out/fused_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "PASS|FAIL|Error|assert" gpurun_out/fused_pytest.log | head -20
for u in 8 16 32; do
  touch paper_2207_11620_b200/csrc/train_tc.cu; make -s -C paper_2207_11620_b200/csrc EXTRA="-DNVOL_AE_CHUNK_U=$u" 2>&1 | grep error
  echo "chunk_u $u"; timeout 120 python tools/fused_diag.py 2>&1 | tail -1
done
