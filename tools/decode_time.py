"""cfg3 decode timing (1024^3 / 1000^3 voxel centres of a cfg2 model), CUDA events.
python tools/decode_time.py [tensor|exact] [dim ...]"""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CFG2, DIMS
from paper_2207_11620_b200.model import build_model
from paper_2207_11620_b200.trainer import decode
m = build_model(CFG2, dims=DIMS, seed=0)
m.infer_mode = sys.argv[1] if len(sys.argv) > 1 else "tensor"
decode(m, dims=(64, 64, 64))
out = []
sizes = [int(a) for a in sys.argv[2:]] or [1024, 1000]
for dims in ((d, d, d) for d in sizes):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f = decode(m, dims=dims); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out.append({"dims": dims[0], "ms": ms, "gsps": dims[0] * dims[1] * dims[2] / ms / 1e6})
    del f
print(json.dumps(out))
