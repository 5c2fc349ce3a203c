#!/usr/bin/env python3
"""Probe (tuning evidence only): can the 1B-edge scaled config (B = 10 GB, DRAM-bound at ~25x
its compulsory bytes) be helped by keeping its hottest B rows in L2?

  a. the plan's fused kernel on the graph as generated (node ids uniformly permuted);
  b. the same sampled SpMM after a degree-sorted relabelling of the columns (B' = B[perm],
     colind' = perm^-1[colind]; every sampled slot maps to the same feature row, per-row slot
     order unchanged -> C bitwise identical), no L2 policy;
  c. (b) with a persisting L2 access-policy window over B's first H rows (the hottest), the rest
     streaming (cuStreamSetAttribute ACCESS_POLICY_WINDOW + CU_LIMIT_PERSISTING_L2_CACHE_SIZE).
L2 flushed before each step, median of 5.  Prints one JSON line per variant."""
import json
import os
import sys

import numpy as np
import torch
from cuda.bindings import driver as cu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402


def main():
    cfg, F, s = "scaled", 256, 128
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph(cfg)
    n = len(rowptr) - 1
    rp = torch.from_numpy(rowptr).to(dev)
    ci = torch.from_numpy(colind).to(dev)
    del colind
    va = torch.ones(ci.numel(), dtype=torch.float32, device=dev)
    B = torch.from_numpy(synth.dense(n, F, synth.seeds(cfg)[1], ld=F)).to(dev)
    C = torch.empty((n, F), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def timed(fn, reps=5):
        ts = []
        for i in range(2 + reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    ms = timed(lambda: es.es_spmm_run(rp, ci, va, B, s, 2, 0, 0, F=F, C=C))
    ref = C.clone()
    print(json.dumps({"variant": "a: as generated", "ms": round(ms, 3)}), flush=True)

    # degree-sorted relabelling of the columns (in-degree = occurrences in colind)
    deg = torch.bincount(ci.long(), minlength=n)
    perm = torch.argsort(deg, descending=True)             # new id -> old id
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(n, device=dev)
    ci2 = inv[ci.long()].to(torch.int32)
    B2 = B[perm].contiguous()
    del B
    ms = timed(lambda: es.es_spmm_run(rp, ci2, va, B2, s, 2, 0, 0, F=F, C=C))
    same = bool(torch.equal(C, ref))
    print(json.dumps({"variant": "b: degree-sorted columns", "ms": round(ms, 3), "bitwise_equal": same}), flush=True)
    cum = torch.cumsum(deg[perm].double(), 0) / deg.sum()

    for hot_mb in (32, 64, 96):
        rows = hot_mb * (1 << 20) // (F * 4)
        (err,) = cu.cuCtxSetLimit(cu.CUlimit.CU_LIMIT_PERSISTING_L2_CACHE_SIZE, hot_mb << 20)
        v = cu.CUstreamAttrValue()
        w = v.accessPolicyWindow
        w.base_ptr = B2.data_ptr()
        w.num_bytes = rows * F * 4
        w.hitRatio = 1.0
        w.hitProp = cu.CUaccessProperty.CU_ACCESS_PROPERTY_PERSISTING
        w.missProp = cu.CUaccessProperty.CU_ACCESS_PROPERTY_STREAMING
        v.accessPolicyWindow = w
        (err2,) = cu.cuStreamSetAttribute(stream.cuda_stream,
                                          cu.CUstreamAttrID.CU_LAUNCH_ATTRIBUTE_ACCESS_POLICY_WINDOW, v)
        ms = timed(lambda: es.es_spmm_run(rp, ci2, va, B2, s, 2, 0, 0, F=F, C=C))
        print(json.dumps({"variant": f"c: + persisting window, hottest {hot_mb} MB", "ms": round(ms, 3),
                          "hot_rows": int(rows), "share_of_endpoints_in_window": round(float(cum[rows - 1]), 4),
                          "bitwise_equal": bool(torch.equal(C, ref)), "cuda_errors": [int(err), int(err2)]}),
              flush=True)
        w.num_bytes = 0
        v.accessPolicyWindow = w
        cu.cuStreamSetAttribute(stream.cuda_stream, cu.CUstreamAttrID.CU_LAUNCH_ATTRIBUTE_ACCESS_POLICY_WINDOW, v)
        cu.cuCtxResetPersistingL2Cache()


if __name__ == "__main__":
    main()
