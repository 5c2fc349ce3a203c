#!/usr/bin/env python3
"""Probe (tuning evidence only): slab-path kernel variants vs the fused kernel, A/B through
es_spmm_options_t.kernel / tune[] (paper_2104_10716_b200.kernel_override).

  python scripts/slab_probe.py [config] [F] [s] [strategy]      # default reddit 602 256 fastrand
  (a fused family -- halfwarp, grouped, ... -- may be listed too: no workspace, no pass timing)
  SLAB_VARIANTS="slab_ldg:4:0:4:0,slab_smem:4:8:4:0"   kernel:stages:width:cta_warps:variant
  UNIFORM_COLS=1: the same degree sequence with uniformly random columns (no popularity skew)
  CONST_DEG=d: nnz/d rows of degree d each, uniform columns (isolates per-row costs)
  NOVAL=1: val = NULL (the unweighted adjacency; no slot values stored or read)
  NOFLUSH=1: no L2 flush between reps (warm L2; F <= 64 then repeats one L2-resident slab)

Each variant: the whole step (L2 flushed before every rep, like bench.py) and the slice passes
alone (reuse_sampled, L2 flushed), median of 8, plus the max difference to the fused kernel's C
and whether it is bitwise equal to the first slab variant.  One JSON line per variant.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402
from bench import byte_model, ldb_for  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 602
    s = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    strat = {"bucket": 1, "fastrand": 2}[sys.argv[4] if len(sys.argv) > 4 else "fastrand"]
    ldb = int(os.environ.get("LDB", ldb_for(F)))
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph(cfg)
    n = len(rowptr) - 1
    K = int(np.minimum(np.diff(rowptr), s).sum())
    Bd = torch.from_numpy(synth.dense(n, F, synth.seeds(cfg)[1], ld=ldb)).to(dev)
    if os.environ.get("UNIFORM_COLS"):        # same degree sequence, columns uniform over [0, n): no popularity skew
        colind = np.random.default_rng(5).integers(0, n, len(colind), dtype=np.int64).astype(np.int32)
    if os.environ.get("CONST_DEG"):           # every row the same degree (isolates per-row costs), uniform columns
        dg = int(os.environ["CONST_DEG"])
        m = len(colind) // dg
        rowptr = (np.arange(m + 1, dtype=np.int64) * dg)
        colind = np.random.default_rng(5).integers(0, n, m * dg, dtype=np.int64).astype(np.int32)
        K = int(np.minimum(np.diff(rowptr), s).sum())
    rp = torch.from_numpy(rowptr).to(dev)
    ci = torch.from_numpy(colind).to(dev)
    va = None if os.environ.get("NOVAL") else torch.ones(len(colind), dtype=torch.float32, device=dev)
    nr = len(rowptr) - 1
    C = torch.zeros((nr, ldb), dtype=torch.float32, device=dev)
    C2 = torch.zeros((nr, ldb), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    bm = byte_model(K, nr, F)
    reps = int(os.environ.get("REPS", 8))

    def timed(fn):
        ts = []
        for i in range(3 + reps):
            if not os.environ.get("NOFLUSH"):
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        return float(np.median(ts)), float(min(ts))

    ms, mn = timed(lambda: es.es_spmm_run_ex(rp, ci, va, Bd, s, strat, 0, 1, F=F, C=C, kernel="fused"))
    print(json.dumps({"config": cfg, "F": F, "s": s, "strategy": strat, "variant": "fused",
                      "plan": es.es_spmm_plan(F, ldb, ldb, Bd, C), "ms": round(ms, 4),
                      "min_ms": round(mn, 4), "algo_GBps": round(bm / ms / 1e6, 1)}), flush=True)
    first = None
    for v in os.environ.get("SLAB_VARIANTS", "slab_ldg,slab_smem").split(","):
        f = v.split(":")
        kern = f[0]
        tune = [int(x) for x in f[1:]] + [0] * (5 - len(f))
        fused_family = kern in ("fused", "warp", "tma", "cpasync", "halfwarp", "rowstream", "grouped", "segstream")
        ws = None if fused_family else es.es_spmm_workspace(nr, n, len(colind), F, ldb, s, va is not None,
                                                            device=dev, kernel=kern)
        C2.zero_()
        kw = dict(F=F, C=C2, workspace=ws, kernel=kern, tune=tune[:4])
        try:
            ms, mn = timed(lambda: es.es_spmm_run_ex(rp, ci, va, Bd, s, strat, 0, 1, **kw))
            pms, pmn = (timed(lambda: es.es_spmm_run_ex(rp, ci, va, Bd, s, strat, 0, 1, reuse_sampled=True, **kw))
                        if ws is not None else (ms, mn))      # fused kernels: no separate passes
        except es.EsError as exc:
            print(json.dumps({"variant": v, "error": str(exc)}), flush=True)
            continue
        st = es.es_spmm_workspace_status(ws) if ws is not None else None
        d = (C2[:, :F] - C[:, :F]).abs().max().item()
        rel = ((C2[:, :F] - C[:, :F]).abs() / C[:, :F].abs().clamp_min(1e-6)).max().item()
        same = None
        if first is None:
            first = C2[:, :F].clone()
        else:
            same = bool(torch.equal(first, C2[:, :F]))
        print(json.dumps({"config": cfg, "F": F, "s": s, "variant": v, "ms": round(ms, 4), "min_ms": round(mn, 4),
                          "passes_ms": round(pms, 4), "passes_min_ms": round(pmn, 4),
                          "algo_GBps": round(bm / ms / 1e6, 1), "ws_status": st,
                          "max_abs_diff_vs_fused": d, "max_rel_diff_vs_fused": rel,
                          "bitwise_eq_first_slab": same}), flush=True)


if __name__ == "__main__":
    main()
