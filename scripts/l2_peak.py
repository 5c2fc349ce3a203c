#!/usr/bin/env python3
"""Measure the L2 ceilings of this B200 (scripts/l2peak.cu) with the clocks sampled during the
run, and write profiles/l2_peak.json -- the roofline denominator bench.py reads for L2-resident
gathers (the slab passes and the fused kernels whose B fits L2).

  python scripts/l2_peak.py [out.json]          # on the GPU box

`l2_stream_gbs` = the best streaming read rate over footprints that fit L2 with room to spare
(<= 96 MB: 32, 48, 60, 64, 80, 96 MB); every probe line is kept under `probes`."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import Clocks  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "l2_peak.json")
    exe = "/tmp/es_l2peak"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-o", exe, os.path.join(ROOT, "scripts", "l2peak.cu")], check=True)
    clocks = Clocks(0)
    clocks.start()
    time.sleep(0.2)
    res = subprocess.run([exe], capture_output=True, text=True, check=True)
    clk = clocks.stop()
    probes = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    stream = [p for p in probes if p.get("probe") == "stream" and p["footprint_MB"] <= 96]
    best = max(stream, key=lambda p: p["GBps"])
    gpu = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.max.sm,clocks.max.mem", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    j = {"l2_stream_gbs": best["GBps"], "footprint_MB": best["footprint_MB"],
         "how": "scripts/l2peak.cu stream_read: every thread streams float4 with ld.global.cg over an L2-resident "
                "footprint (4 x 512-thread CTAs per SM), best of 5 timed launches of ~8 GiB each (CUDA events); "
                "best over footprints <= 96 MB",
         "gpu": gpu, "clocks": clk, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "probes": probes}
    with open(out, "w") as f:
        json.dump(j, f, indent=1)
    print(json.dumps({k: j[k] for k in ("l2_stream_gbs", "footprint_MB", "clocks")}))


if __name__ == "__main__":
    main()
