"""profiles/<tag>_ncu_summary.md -> profiles/ncu_traffic.json (per-kernel DRAM bytes per launch,
read by bench.py for roofline.traffic).   python tools/ncu_traffic.py r1d"""
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
s = (ROOT / "profiles" / f"{tag}_ncu_summary.md").read_text()
out = {}
for sec in re.split(r"\n### ", s)[1:]:
    name = re.sub(r"<.*", "", re.sub(r"^void ", "", sec.split("\n")[0].strip()))
    rd = re.search(r"DRAM read: ([0-9.]+) Mbyte", sec)
    wr = re.search(r"DRAM write: ([0-9.]+) Mbyte", sec)
    du = re.search(r"duration: ([0-9.]+) us", sec)
    if rd and wr and name not in out:
        out[name] = {"dram_read_mb": float(rd.group(1)), "dram_write_mb": float(wr.group(1)),
                     "traffic_bytes": (float(rd.group(1)) + float(wr.group(1))) * 1e6,
                     "ncu_duration_us": float(du.group(1)) if du else None}
out["_source"] = (f"profiles/{tag}_ncu_summary.md: one ncu --set full --cache-control none --clock-control none "
                  f"capture per kernel (tools/gpu_round_evidence.sh {tag})")
(ROOT / "profiles" / "ncu_traffic.json").write_text(json.dumps(out, indent=1))
print(json.dumps({k: v["traffic_bytes"] for k, v in out.items() if k != "_source"}))
