#!/usr/bin/env python3
"""Copy a measurement pass (scripts/gpu_r01j.sh <tag> -> gpurun_out/<tag>/) into profiles/ and
regenerate the measured tables of BASELINE.md and README.md (between their <!-- x:begin/end -->
markers) from those JSON lines.  Usage: python scripts/update_tables.py gpurun_out/r01q"""
import json
import os
import re
import shutil
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
CFG = [("**Reddit F=602, s=256, FastRand, mean (graded)**", "reddit602"), ("Reddit F=128, s=256, FastRand, mean", "reddit128"),
       ("Proteins F=128, s=256, FastRand, sum", "proteins"), ("Arxiv F=128, s=64, FastRand, sum", "arxiv"),
       ("Pubmed F=16, s=32, Bucket, sum", "pubmed"), ("Scaled 10M / 1.0B, F=256, s=128, FastRand, sum", "scaled")]


def replace(path, tag, body):
    s = open(path).read()
    s = re.sub(rf"<!-- {tag}:begin -->\n.*?\n<!-- {tag}:end -->", f"<!-- {tag}:begin -->\n{body}\n<!-- {tag}:end -->",
               s, flags=re.S)
    open(path, "w").write(s)


def main():
    src = sys.argv[1]
    for _, n in CFG:
        shutil.copy(os.path.join(src, f"bench_{n}.json"), os.path.join(P, f"r01_bench_{n}.json"))
    shutil.copy(os.path.join(src, "ref_reddit602.json"), os.path.join(P, "r01_ref_reddit602.json"))
    shutil.copy(os.path.join(src, "launches_reddit602.csv"), os.path.join(P, "r01_launches_reddit_f602.csv"))
    for n in ("reddit602", "reddit128", "proteins"):
        for a, b in ((f"step_{n}.json", f"r01_ncu_step_{n}.json"), (f"step_{n}.summary.jsonl", f"r01_ncu_full_step_{n}.jsonl")):
            if os.path.exists(os.path.join(src, a)):
                shutil.copy(os.path.join(src, a), os.path.join(P, b))
    for a, b in (("s_sweep.jsonl", "r01_s_sweep.jsonl"), ("e2e_gnn.jsonl", "r01_e2e_gnn_reddit.jsonl")):
        if os.path.exists(os.path.join(src, a)) and os.path.getsize(os.path.join(src, a)) > 0:
            shutil.copy(os.path.join(src, a), os.path.join(P, b))
    rows, rrows = [], []
    for name, n in CFG:
        d = json.load(open(os.path.join(P, f"r01_bench_{n}.json")))
        r, st = d["roofline"], d["roofline"].get("step")
        kern = ("`spmm_slab` ×%d + sampling" % r["launches_per_step"]) if st else \
            "`%s`" % r["kernel"].replace("es::", "").split("(")[0]
        frac = f"{r['frac']:.2f} (step {st['frac']:.2f})" if st else f"{r['frac']:.2f}"
        K = d["config"]["K_sampled"]
        rows.append(f"| {name} | {K / 1e6:.2f}M | {d['ms_per_step']:.3f} ({d['detail']['step_ms_min']:.3f}) | "
                    f"{d['value']:,.0f} | {r['achieved']:,.0f} | {frac} | {d['e2e']['value']:,.0f} | "
                    f"{d['cpu_baseline']['value']:.1f} | {kern} |")
        rrows.append(f"| {d['config']['workload']} | {d['ms_per_step']:.3f} | {d['value']:,.0f} | "
                     f"{r['achieved']:,.0f} ({r['frac']:.2f}) |")
    hdr = ("| config | K sampled | ms / step | GFLOP/s | model GB/s | frac of 6548 GB/s | e2e GFLOP/s (host buffers) "
           "| oracle, 16 cores | kernel |\n|---|---|---|---|---|---|---|---|---|\n")
    replace(os.path.join(ROOT, "BASELINE.md"), "measured", hdr + "\n".join(rows))
    replace(os.path.join(ROOT, "README.md"), "readme", "| workload | ms / step (median) | GFLOP/s | dominant kernel's "
            "algorithmic GB/s (× of 6.55 TB/s copy BW) |\n|---|---|---|---|\n" + "\n".join(rrows))
    sw = os.path.join(P, "r01_s_sweep.jsonl")
    t = defaultdict(dict)
    for line in open(sw):
        x = json.loads(line)
        t[(x["graph"], x["F"], x["reduce"])][(x["s"], x["strategy"])] = x
    lines = ["| graph, F, reduce | s=16 | 32 | 64 | 128 | 256 | 512 |", "|---|---|---|---|---|---|---|"]
    for (g, F, red), dd in t.items():
        cells = []
        for s in (16, 32, 64, 128, 256, 512):
            b, f = dd[(s, "bucket")], dd[(s, "fastrand")]
            mark = " †" if "slab" in b["plan"] else ""
            cells.append(f"{b['GFLOPs']:,.0f} ({b['frac']:.2f}) / {f['GFLOPs']:,.0f} ({f['frac']:.2f}){mark}")
        lines.append(f"| {g}, {F}, {red} | " + " | ".join(cells) + " |")
    replace(os.path.join(ROOT, "BASELINE.md"), "ssweep", "\n".join(lines))
    print("\n".join(rows))


if __name__ == "__main__":
    main()
