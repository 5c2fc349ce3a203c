#!/usr/bin/env python3
"""Summarise an .ncu-rep (raw page) into the metrics this repo reports."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct_peak",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "smsp__inst_executed.sum": "inst",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__t_bytes.sum": "l1_bytes",
}


def to_bytes(v, unit):
    f = float(v)
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit)
    return f * mul if mul else f


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for i, h in enumerate(hdr):
            if h in WANT:
                u = units[i]
                if "byte" in u:
                    d[WANT[h]] = to_bytes(vals[i], u)
                elif u == "ms":
                    d[WANT[h]] = float(vals[i]) * 1e-3
                elif u == "us":
                    d[WANT[h]] = float(vals[i]) * 1e-6
                elif u == "ns":
                    d[WANT[h]] = float(vals[i]) * 1e-9
                else:
                    try:
                        d[WANT[h]] = float(vals[i])
                    except ValueError:
                        d[WANT[h]] = vals[i]
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["top_stalls"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:5]}
        if "duration" in d and "dram_read" in d:
            d["dram_GBs"] = (d["dram_read"] + d.get("dram_write", 0)) / d["duration"] / 1e9
        out.append(d)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summarise(p):
            print(json.dumps({"file": p, **d}))
