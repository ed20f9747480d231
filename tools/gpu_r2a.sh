# round 2 first check: full GPU suite, bench, source-level ncu of the MLP kernel
export PYTHONUNBUFFERED=1
tag=${1:-r2a}
timeout 1200 python -m pytest tests -m gpu -q -rs --timeout 900 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_$tag.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo bench=$?; tail -c 600 gpurun_out/bench_$tag.log
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"mlp_tc" -s 2 -c 1 -o gpurun_out/prof_mlp_$tag python tools/prof_step.py --steps 3 > gpurun_out/ncu_$tag.log 2>&1; echo prof=$?
