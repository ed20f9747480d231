export PYTHONUNBUFFERED=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_simt.csv python tools/prof_step.py --mode 0 --steps 3 > /dev/null 2>&1
python tools/launches2.py gpurun_out/launches_simt.csv 40 | tail -30
NVOL_DETERMINISTIC=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_det.csv python -c "
import sys; sys.path.insert(0,'.'); sys.argv=['x','--mode','0','--steps','3']
from paper_2207_11620_b200 import encoding; encoding.set_deterministic(True)
exec(open('tools/prof_step.py').read())
" > /dev/null 2>&1
python tools/launches2.py gpurun_out/launches_det.csv 40 | tail -30
