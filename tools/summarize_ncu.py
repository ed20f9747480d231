"""Summarise ncu captures (--set full) + a launch list into profiles/<tag>_*.md.

    python tools/summarize_ncu.py <tag> <launches.csv> <rep> [<rep> ...]
"""
import csv
import io
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "tcgen05 fp16 tensor ops % of peak"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor-memory path active %"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 RED requests"),
    ("lts__t_requests_srcunit_tex_op_read.sum", "L2 read requests"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m, label in METRICS:
            if m in hdr:
                d[label] = (r[hdr.index(m)], units[hdr.index(m)])
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x)
                  for h, x in zip(hdr, r) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h.endswith("not_issued") and x.replace(".", "", 1).isdigit()}
        tot = sum(stalls.values()) or 1.0
        d["top stalls"] = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in
                                    sorted(stalls.items(), key=lambda kv: -kv[1])[:4])
        res.append(d)
    return res


def main():
    tag, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = [f"# ncu summary — {tag}", ""]
    lines += ["## Launch list (warm cache, serialised; `--cache-control none --clock-control none`)", "",
              "```"]
    lines += subprocess.run([sys.executable, str(ROOT / "tools" / "launches2.py"), launches, "12"],
                            capture_output=True, text=True).stdout.rstrip().splitlines()
    lines += ["```", ""]
    for rep in reps:
        lines += [f"## `{Path(rep).name}` (`--set full`)", ""]
        for d in raw(rep):
            lines.append(f"### {d.pop('kernel')}")
            for k, v in d.items():
                if isinstance(v, tuple):
                    lines.append(f"- {k}: {v[0]} {v[1]}")
                else:
                    lines.append(f"- {k}: {v}")
            lines.append("")
    out = ROOT / "profiles" / f"{tag}_ncu_summary.md"
    out.write_text("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main()
