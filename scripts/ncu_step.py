#!/usr/bin/env python3
"""Aggregate an ncu --set full report of ONE bench step (all of its launches) into per-kernel
and per-step DRAM traffic / duration (tuning evidence; feeds profiles/ncu_traffic.json)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarise  # noqa: E402


def main():
    rows = summarise(sys.argv[1])
    tot_t = sum(r.get("duration", 0.0) for r in rows)
    tot_b = sum(r.get("dram_read", 0.0) + r.get("dram_write", 0.0) for r in rows)
    by = {}
    for r in rows:
        k = r["kernel"].split("(")[0]
        d = by.setdefault(k, {"launches": 0, "duration_s": 0.0, "dram_bytes": 0.0})
        d["launches"] += 1
        d["duration_s"] += r.get("duration", 0.0)
        d["dram_bytes"] += r.get("dram_read", 0.0) + r.get("dram_write", 0.0)
    for d in by.values():
        d["share_of_step_time"] = round(d["duration_s"] / tot_t, 4) if tot_t else None
    print(json.dumps({"file": sys.argv[1], "launches": len(rows), "step_duration_s_serialised": tot_t,
                      "step_dram_bytes": tot_b, "kernels": by}))


if __name__ == "__main__":
    main()
