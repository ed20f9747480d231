export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_render.py -q -p no:cacheprovider > gpurun_out/render_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/render_pytest.log; grep -E "^E " gpurun_out/render_pytest.log | head -10
timeout 300 python - <<'PY'
import time, torch, sys
sys.argv = ["x", "tensor"]
exec(open("tools/prof_render.py").read().replace("torch.cuda.profiler.start()", "pass").replace("torch.cuda.profiler.stop()", "pass"))
for mode in ("tensor", "exact"):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); a = time.perf_counter()
        img, st = render_frame_device(m, tf, cam, cfg, grid, "wavefront", mode)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - a) * 1e3)
    print(mode, "frame ms", [round(t, 3) for t in sorted(ts)], st.evals, len(st.alive_per_iteration))
PY
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/render_launches_warm.csv python tools/prof_render.py tensor 2>&1 | grep -v "^==PROF==" | tail -1
python tools/summ_launch.py gpurun_out/render_launches_warm.csv
