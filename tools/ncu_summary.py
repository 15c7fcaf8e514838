"""Summarise ncu --set full captures (.ncu-rep) into the committed profiles/ text + the per-launch DRAM
traffic JSON bench.py reads for roofline.traffic.

    python tools/ncu_summary.py TAG   # reads gpurun_out/TAG_{lu,sweep,spmv}.ncu-rep and TAG_launches_C.csv
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import launches  # noqa: E402

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active % (active SMs)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier /issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard /issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard /issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait /issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle /issue"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {name: (val, unit) for name, unit, val in zip(h, u, v)}, v[h.index("Kernel Name")]


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(val.replace(",", "")) * scale.get(unit, 1)


def main(tag):
    out_dir = os.path.join(ROOT, "profiles")
    lines = [f"# ncu summaries ({tag}): one launch each, --set full --clock-control none (cold caches, serialised)", ""]
    traffic = {}
    for part in ("lu", "luD", "sweep", "spmv", "spmv2"):
        rep = os.path.join(ROOT, "gpurun_out", f"{tag}_{part}.ncu-rep")
        if not os.path.exists(rep):
            continue
        d, name = raw(rep)
        lines.append(f"## {part}: {name[:110]}")
        for key, label in KEYS:
            if key in d:
                val, unit = d[key]
                lines.append(f"  {label:38s} {val} {unit}")
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if rd and wr:
            tb = to_bytes(*rd) + to_bytes(*wr)
            lines.append(f"  {'DRAM read+write per launch':38s} {tb / 1e9:.4f} GB")
            traffic[part] = tb
        lines.append("")
    lc = os.path.join(ROOT, "gpurun_out", f"{tag}_launches_C.csv")
    if os.path.exists(lc):
        lines.append("## launch list (bench.py --steps 1 --warmup 1, SaP-C; gpu__time_duration per kernel)")
        lines.append(launches.summarise(lc))
    ld = os.path.join(ROOT, "gpurun_out", f"{tag}_launches_D.csv")
    if os.path.exists(ld):
        lines.append("")
        lines.append("## launch list (bench.py --precond D --steps 1 --warmup 1, SaP-D)")
        lines.append(launches.summarise(ld))
    with open(os.path.join(out_dir, f"ncu_{tag}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if "lu" in traffic:
        with open(os.path.join(out_dir, "ncu_lu_traffic.json"), "w") as f:
            json.dump({"SaP-C": traffic["lu"], "SaP-D": traffic.get("luD"),
                       "source": f"profiles/ncu_{tag}.txt (dram__bytes_read.sum + dram__bytes_write.sum of one "
                       "band LU launch (k_band_lu_df) of config 2: LU+UL for SaP-C (lu), LU for SaP-D (luD))",
                       "sweep": traffic.get("sweep"), "spmv": traffic.get("spmv")}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1])
