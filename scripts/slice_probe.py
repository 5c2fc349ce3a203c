#!/usr/bin/env python3
"""Probe (tuning evidence only): does feature slicing make the B gathers L2-resident?

Reddit-shaped graph, F=602 (ldb 608).  Compares, per step (L2 flushed before each):
  fused  : one es_spmm_run over the full width (the plan's kernel)
  sliced : es_spmm_sample (compact slot-order CSR of the sampled edges) + one es_spmm_run per
           feature slice [c0, c0+w) over that compact CSR (Bucket, s = inf: takes every slot in
           slot order, i.e. the same sampled SpMM), so each pass gathers a B slice of
           N * w * 4 bytes -- L2-resident for w <= ~96.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402
from bench import byte_model  # noqa: E402


def main():
    F, ldb, s = 602, 608, 256
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph("reddit")
    n = len(rowptr) - 1
    K = int(np.minimum(np.diff(rowptr), s).sum())
    Bd = torch.from_numpy(synth.dense(n, F, synth.seeds("reddit")[1], ld=ldb)).to(dev)
    rp = torch.from_numpy(rowptr).to(dev)
    ci = torch.from_numpy(colind).to(dev)
    va = torch.ones(len(colind), dtype=torch.float32, device=dev)
    C = torch.zeros((n, ldb), dtype=torch.float32, device=dev)
    C2 = torch.zeros((n, ldb), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lib = es.load_library()
    st = torch.cuda.current_stream().cuda_stream
    srp, sci, sva, _ = es.es_spmm_sample(rp, ci, va, s, 2, 0, want_pos=False)

    def timed(fn, reps=6):
        ts = []
        for i in range(2 + reps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        return float(np.median(ts)), float(min(ts))

    def fused():
        es.es_spmm_run(rp, ci, va, Bd, s, 2, 0, 1, F=F, C=C)

    def materialize():
        rc = lib.es_spmm_sample(n, n, rp.data_ptr(), ci.data_ptr(), va.data_ptr(), s, 2, 0, 0,
                                srp.data_ptr(), sci.data_ptr(), sva.data_ptr(), None, st)
        assert rc == 0

    def passes(w):
        def go():
            for c0 in range(0, F, w):
                wf = min(w, F - c0)
                rc = lib.es_spmm_run(n, n, srp.data_ptr(), sci.data_ptr(), sva.data_ptr(),
                                     Bd.data_ptr() + 4 * c0, wf, ldb, 1 << 30, 1, 0, 1,
                                     C2.data_ptr() + 4 * c0, ldb, st)
                assert rc == 0
        return go

    bm = byte_model(K, n, F)
    ms, mn = timed(fused)
    print(json.dumps({"variant": "fused", "plan": es.es_spmm_plan(F, ldb, ldb, Bd, C), "ms": round(ms, 3),
                      "min_ms": round(mn, 3), "algo_GBps": round(bm / ms / 1e6, 1)}), flush=True)
    ms_m, _ = timed(materialize)
    print(json.dumps({"variant": "materialize", "ms": round(ms_m, 3)}), flush=True)
    variants = [(w, {}) for w in [64, 128, 304]]
    variants += [(w, {"ES_SPMM_CPASYNC_MIN_NV4": "4", "ES_SPMM_STAGES": st})
                 for w in [32, 48, 64, 96] for st in ["4", "8"]]
    for w, env in variants:
        for k in [k for k in os.environ if k.startswith("ES_SPMM_")]:
            os.environ.pop(k)
        os.environ.update(env)
        go = passes(w)
        ms, mn = timed(go)
        torch.cuda.synchronize()
        d = (C2[:, :F] - C[:, :F]).abs().max().item()
        print(json.dumps({"variant": f"sliced w={w}", "env": env, "plan": es.es_spmm_plan(min(w, F), ldb, ldb, Bd, C2),
                          "passes_ms": round(ms, 3), "min_ms": round(mn, 3),
                          "with_materialize_ms": round(ms + ms_m, 3),
                          "algo_GBps": round(bm / (ms + ms_m) / 1e6, 1), "max_abs_diff_vs_fused": d}),
              flush=True)


if __name__ == "__main__":
    main()
