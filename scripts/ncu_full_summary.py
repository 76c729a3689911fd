"""Summarise `ncu -i <rep> --page raw --csv` exports of single-kernel captures into the JSON
bench.py reads for the roofline `traffic` (dram bytes per launch) and the per-kernel evidence.

usage: python scripts/ncu_full_summary.py "key|shape|path.csv" [...] > profiles/r1_ncu_full_kernels.json"""
import csv
import json
import sys

WANT = {
    "time_us_cold": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l2_hit_rate_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "imma_inst_pct_active": ("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active", 1.0),
    "mem_tensor_pct_active": ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
}
UNIT = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9,
        "%": 1.0}


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, units, data = rows[h], rows[h + 1], rows[h + 2:]
    last = data[-1]                         # the captured launch (one per report)
    col = {n: i for i, n in enumerate(hdr)}
    rec = {"kernel": last[col["Kernel Name"]], "grid": last[col.get("Grid Size", 0)]}
    for key, (metric, scale) in WANT.items():
        i = col.get(metric)
        if i is None or not last[i]:
            continue
        v = float(last[i].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            v = v * UNIT.get(units[i], 1.0) * 1e-3      # -> us
        elif "bytes" in metric:
            v = v * UNIT.get(units[i], 1.0)
        rec[key] = v
    if "dram_read_bytes" in rec:
        rec["traffic_bytes"] = rec["dram_read_bytes"] + rec.get("dram_write_bytes", 0.0)
    return rec


out = {}
for arg in sys.argv[1:]:
    key, shape, path = arg.split("|")
    rec = load(path)
    rec["shape"] = shape
    out[key] = rec
print(json.dumps(out, indent=1))
