#!/usr/bin/env python3
"""Interleaved A/B of the per-B-row L2 residency hint (es_spmm_options_t.b_hot_mask).

Hot set = the B rows gathered most often by the sampled graph (exact access counts from
es_spmm_sample), largest first, up to a byte budget; variants are timed round-robin
(flush, launch) so clock/thermal drift hits all of them alike.  Tuning evidence only."""
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
    name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 602
    s = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    budgets = [int(x) for x in (sys.argv[4] if len(sys.argv) > 4 else "0,30,50,70,90,110").split(",")]
    rounds = 8
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph(name)
    n = len(rowptr) - 1
    ldb = ldb_for(F)
    B = torch.from_numpy(synth.dense(n, F, synth.seeds(name)[1], ld=ldb)).to(dev)
    rp, ci = torch.from_numpy(rowptr).to(dev), torch.from_numpy(colind).to(dev)
    va = torch.ones(len(colind), device=dev)
    C = torch.empty((n, ldb), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    _, sc, _, _ = es.es_spmm_sample(rp, ci, va, s, 2, 0, want_pos=False)
    counts = torch.bincount(sc.long(), minlength=n).cpu().numpy()
    order = np.argsort(-counts, kind="stable")
    row_bytes = ldb * 4
    masks = {}
    for mb in budgets:
        if mb == 0:
            masks[mb] = None
            continue
        top = order[: int(mb * 1e6 // row_bytes)]
        bits = np.zeros((n + 31) // 32, dtype=np.uint32)
        np.bitwise_or.at(bits, top >> 5, (np.uint32(1) << (top & 31).astype(np.uint32)))
        frac = counts[top].sum() / counts.sum()
        masks[mb] = (torch.from_numpy(bits.view(np.int32)).to(dev), float(frac))
    K = int(counts.sum())
    ts = {mb: [] for mb in budgets}
    for r in range(rounds + 1):
        for mb in budgets:
            m = masks[mb]
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            es.es_spmm_run_ex(rp, ci, va, B, s, 2, 0, 1, F=F, C=C, hot_mask=None if m is None else m[0])
            e1.record()
            torch.cuda.synchronize()
            if r > 0:
                ts[mb].append(e0.elapsed_time(e1))
    for mb in budgets:
        ms = float(np.median(ts[mb]))
        print(json.dumps({"graph": name, "F": F, "s": s, "hot_budget_MB": mb,
                          "hot_access_frac": None if masks[mb] is None else round(masks[mb][1], 3),
                          "ms_median": round(ms, 3), "ms_min": round(min(ts[mb]), 3),
                          "model_TBs": round(byte_model(K, n, F) / (ms / 1e3) / 1e12, 2),
                          "plan": es.es_spmm_plan(F, ldb, ldb, B, C)}), flush=True)


if __name__ == "__main__":
    main()
