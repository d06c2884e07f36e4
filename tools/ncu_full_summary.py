"""Summarize an `ncu --set full` report (exported with `ncu -i X.ncu-rep --page raw --csv`) into JSON.

    python tools/ncu_full_summary.py raw.csv out.json "source description"
Keeps, per launch: kernel, duration, DRAM bytes read/written, DRAM throughput %, achieved occupancy, registers and
the main stall ratios.  The bench's roofline `traffic` field reads `dram_bytes_read + dram_bytes_write` from here.
"""
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "msecond": 1e3,
         "usecond": 1.0, "nsecond": 1e-3}


def col(r, name, conv=float):
    if name not in hdr:
        return None
    i = hdr.index(name)
    v = r[i].replace(",", "")
    try:
        x = conv(v)
    except ValueError:
        return v
    return x * SCALE.get(units[i], 1.0) if conv is float else x


def key(name):
    base = re.sub(r"\(.*", "", name).replace("void ", "")
    base = re.sub(r"^fpd::", "", base)
    m = re.match(r"(\w+)(<.*>)?", base)
    k = m.group(1).replace("_kernel", "")
    ep = re.findall(r"E[A-Z]\w+", name)
    return k + ("_" + ep[0] if ep else "")


out = {"source": sys.argv[3] if len(sys.argv) > 3 else "", "kernels": {}}
for r in data:
    name = col(r, "Kernel Name", str)
    k = key(name)
    i = 2
    while k in out["kernels"]:
        k = f"{key(name)}#{i}"
        i += 1
    out["kernels"][k] = {
        "kernel": name,
        "grid": col(r, "Grid Size", str),
        "gpu_time_us": col(r, "gpu__time_duration.sum"),
        "dram_bytes_read": col(r, "dram__bytes_read.sum"),
        "dram_bytes_write": col(r, "dram__bytes_write.sum"),
        "dram_throughput_pct": col(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_pct": col(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": col(r, "launch__registers_per_thread", str),
        "stall_long_scoreboard_per_issue": col(
            r, "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
        "stall_barrier_per_issue": col(r, "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"),
    }
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps({k: (v["gpu_time_us"], v["dram_bytes_read"]) for k, v in out["kernels"].items()}, indent=0))
