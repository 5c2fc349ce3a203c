#!/usr/bin/env python3
"""profiles/ncu_traffic.json from a measurement pass (scripts/gpu_pass.sh): per config, the ncu
DRAM bytes (read + write) per launch of the dominant kernel, averaged over its launches of one
step -- bench.py reports them as roofline.traffic / dram_frac.

  python scripts/traffic_table.py gpurun_out/<tag> <tag>"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# capture name -> bench key (config|F|s|strategy|reduce[|slab])
KEYS = {"reddit602": "reddit|F602|s256|fastrand|mean|slab", "reddit128": "reddit|F128|s256|fastrand|mean|slab",
        "proteins": "proteins|F128|s256|fastrand|sum|slab", "arxiv": "arxiv|F128|s64|fastrand|sum",
        "pubmed": "pubmed|F16|s32|bucket|sum", "scaled": "scaled|F256|s128|fastrand|sum"}


def main():
    d, tag = sys.argv[1], sys.argv[2]
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    for name, key in KEYS.items():
        f = os.path.join(d, f"prof_{name}.summary.jsonl")
        if not os.path.exists(f):
            continue
        rows = [json.loads(x) for x in open(f) if x.strip().startswith("{")]
        rows = [r for r in rows if "dram_read" in r]
        if not rows:
            continue
        per = [r["dram_read"] + r.get("dram_write", 0.0) for r in rows]
        dur = sum(r["duration"] for r in rows)
        table[key] = {"dram_bytes_per_launch": int(sum(per) / len(per)), "launches": len(rows),
                      "kernel": rows[0]["kernel"], "l2_hit_pct": round(sum(r["l2_hit_pct"] for r in rows) / len(rows), 2),
                      "dram_GBs_under_ncu": round(sum(per) / dur / 1e9),
                      "source": f"profiles/{tag}_ncu_full_{name}.jsonl (ncu --set full, the dominant kernel's "
                                f"{len(rows)} launch(es) of one step)"}
        os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_{name}.jsonl"), "w") as fo:
            fo.writelines(json.dumps(r) + "\n" for r in rows)
    with open(path, "w") as fo:
        json.dump(table, fo, indent=1)
    print(json.dumps({k: v["dram_bytes_per_launch"] for k, v in table.items()}))


if __name__ == "__main__":
    main()
