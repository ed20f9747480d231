export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_i.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu_i.log
for v in 0 100000000; do
  NVOL_L2_PERSIST=$v timeout 600 python bench.py --no-cpu --no-decode --no-render > gpurun_out/bench_i$v.log 2>&1; echo bench$v=$?; tail -1 gpurun_out/bench_i$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
  NVOL_L2_PERSIST=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_i$v.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1
done
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('l2', p.L2_cache_size)
from paper_2207_11620_b200 import _lib; print('persist max ->', _lib.load().nvol_l2_persist(1<<40))"
