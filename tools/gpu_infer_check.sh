export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_render.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "render or tensor_inference or decode" > gpurun_out/infer_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/infer_pytest.log
timeout 600 python bench.py --no-cpu --no-cfg5 2>&1 | tail -1 > gpurun_out/bench_infer.json
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_infer.json"))
print("train", d["value"], d["ms_per_step"])
print("decode", d["decode"]["value"], d["decode"]["ms"])
r = d["render"]
for k in ("wavefront_tensor", "wavefront_exact", "inshader_exact"):
    print(k, r[k]["frame_ms"], r[k]["evals_per_s"], r[k]["iterations"])
PY
