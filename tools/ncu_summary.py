"""Summarise ncu reports (run here, on the CPU side) into profiles/.

  python tools/ncu_summary.py <report.ncu-rep> [...]    -> prints a markdown table
  python tools/ncu_summary.py --launches launches.csv    -> per-kernel launch-time shares
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (realtime)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor memory active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster x"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    for r in rows[2:]:
        res.append(dict(zip(rows[0], r)) | {"_units": dict(zip(rows[0], rows[1]))})
    return res


def stalls(d, n=6):
    st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v))
          for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and
          k.endswith("_per_issue_active.ratio") and v not in ("", None)]
    st.sort(key=lambda x: -x[1])
    return st[:n]


def summarize(rep):
    lines = []
    for d in raw(rep):
        u = d["_units"]
        lines.append(f"### `{d.get('Kernel Name', '?')[:110]}`\n")
        lines.append("| metric | value |\n|---|---|")
        for k, name in KEYS:
            if k in d and d[k] != "":
                lines.append(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        lines.append("\nTop warp stall reasons (cycles per issued instruction): " +
                     ", ".join(f"{k} {v:.2f}" for k, v in stalls(d)) + "\n")
    return "\n".join(lines)


def traffic(rep):
    d = raw(rep)[0]
    mb = float(d["dram__bytes_read.sum"]) if d["_units"]["dram__bytes_read.sum"] == "Mbyte" else None
    rd = float(d["dram__bytes_read.sum"]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[d["_units"]["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[d["_units"]["dram__bytes_write.sum"]]
    return rd + wr


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    acc = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            acc[r[ki]].append(float(r[vi].replace(",", "")))
    return acc


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        acc = launches(sys.argv[2])
        tot = sum(sum(v) for v in acc.values())
        print("| kernel | launches | mean ns | share of listed time |\n|---|---|---|---|")
        for k, v in sorted(acc.items(), key=lambda x: -sum(x[1])):
            print(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v):.0f} | {sum(v) / tot:.3f} |")
    elif sys.argv[1] == "--traffic":
        print(json.dumps({"bytes": traffic(sys.argv[2])}))
    else:
        for rep in sys.argv[1:]:
            print(summarize(rep))
