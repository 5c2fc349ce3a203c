#!/usr/bin/env python3
"""NEXT-3: the fused sampled SpMM vs cuSPARSE on the same B200.

The paper's baseline is cusparseSpMM on the full graph (L1268) and, in §5.6 (L1509-1524),
cuSPARSE fed a pre-sampled graph.  For the Reddit-shaped graph and several s:
  exact      : cuSPARSE CSR SpMM (torch.sparse, int32 indices) on the full A
  presampled : es_spmm_sample (materialised sampled CSR, slot order) -> cuSPARSE SpMM
               (timed as sample + SpMM and SpMM alone)
  fused      : es_spmm_run (sampling inside the kernel)
L2 flushed before every timed call, CUDA events, median of 5.  Prints JSON lines."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402


def timeit(fn, flush, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 602
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph(name)
    n = len(rowptr) - 1
    ldb = (F + 3) // 4 * 4
    Bp = torch.from_numpy(synth.dense(n, F, synth.seeds(name)[1], ld=ldb)).to(dev)
    Bc = Bp[:, :F].contiguous()                   # cuSPARSE gets a dense n x F operand
    rp = torch.from_numpy(rowptr).to(dev)
    ci = torch.from_numpy(colind).to(dev)
    va = torch.ones(len(colind), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    A = torch.sparse_csr_tensor(rp.to(torch.int32), ci, va, size=(n, n))
    t_exact = timeit(lambda: A @ Bc, flush)
    print(json.dumps({"graph": name, "F": F, "case": "exact cuSPARSE", "ms": round(t_exact, 3)}), flush=True)
    C = torch.empty((n, ldb), dtype=torch.float32, device=dev)
    for strat, s in [(1, 16), (2, 16), (1, 32), (2, 32), (2, 64), (2, 256)]:
        t_fused = timeit(lambda: es.es_spmm_run(rp, ci, va, Bp, s, strat, 0, 0, F=F, C=C), flush)
        srp, sc, sv, _ = es.es_spmm_sample(rp, ci, va, s, strat, 0, want_pos=False)
        As = torch.sparse_csr_tensor(srp.to(torch.int32), sc, sv, size=(n, n))
        t_spmm = timeit(lambda: As @ Bc, flush)

        def pre():
            r, c, v, _ = es.es_spmm_sample(rp, ci, va, s, strat, 0, want_pos=False)
            return torch.sparse_csr_tensor(r.to(torch.int32), c, v, size=(n, n)) @ Bc
        t_pre = timeit(pre, flush)
        ref = (As @ Bc)
        got = C[:, :F]
        rel = float(((got - ref).abs() / ref.abs().clamp_min(1e-6)).max())
        print(json.dumps({"graph": name, "F": F, "strategy": "bucket" if strat == 1 else "fastrand", "s": s,
                          "fused_ms": round(t_fused, 3), "presampled_cusparse_spmm_ms": round(t_spmm, 3),
                          "presampled_sample_plus_spmm_ms": round(t_pre, 3), "exact_cusparse_ms": round(t_exact, 3),
                          "speedup_fused_vs_exact": round(t_exact / t_fused, 2),
                          "speedup_fused_vs_presampled_spmm": round(t_spmm / t_fused, 2),
                          "max_rel_diff_fused_vs_cusparse": rel}), flush=True)


if __name__ == "__main__":
    main()
