#!/usr/bin/env python3
"""Small calls of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck).  Run: compute-sanitizer --tool memcheck python scripts/sanitize.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402


def main():
    dev = "cuda:0"
    rowptr, colind, val = synth.random_csr(300, 700, seed=2, max_deg=150, special=(577, 600, 0))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    rp, ci, va = t(rowptr), t(colind), t(val)
    cases = [(16, 16, None), (41, 44, None), (128, 128, None), (200, 200, "tma"), (256, 256, None),
             (602, 604, None), (602, 602, None), (1100, 1100, None), (130, 130, "warp")]
    for F, ldb, kern in cases:
        B = t(synth.dense(700, F, seed=F, ld=ldb))
        with es.kernel_override(kern or "auto"):
            for strat in (1, 2):
                for red in (0, 1):
                    C = es.es_spmm_run(rp, ci, va, B, 64, strat, 5, red, F=F)
        torch.cuda.synchronize()
        print("ok", F, ldb, es.es_spmm_plan(F, ldb, F, B, C), flush=True)
    # slab path (forced): every slab kernel, narrow tails, and a workspace sized for a quarter of
    # the stored entries with that nnz stated (the device backstop poisons the rows that do not fit)
    for fam, tune in (("slab_smem", (0, 8)), ("slab_smem", (0, 16)), ("slab_ldg", ()), ("slab_tma", ())):
        with es.kernel_override(fam, *tune):
            for F, ldb in ((602, 608), (130, 136), (200, 200), (17, 24)):
                B = t(synth.dense(700, F, seed=F, ld=ldb))
                for nnz in (len(colind), len(colind) // 4):
                    ws = es.es_spmm_workspace(300, 700, nnz, F, ldb, 64, True, device=dev)
                    for strat in (1, 2):
                        es.es_spmm_run_ex(rp, ci, va, B, 64, strat, 5, 1, F=F, workspace=ws, nnz=nnz)
                    es.es_spmm_run_ex(rp, ci, None, B, 64, 2, 5, 0, F=F, workspace=ws, nnz=nnz)
                    es.es_spmm_run_ex(rp, ci, va, B, 64, 2, 5, 1, F=F, workspace=ws, reuse_sampled=True, nnz=nnz)
                torch.cuda.synchronize()
                print("ok slab", fam, tune, F, ldb, flush=True)
    # bf16 storage on the slab path (128-element slices + narrow tails) and the slab backward
    with es.kernel_override("slab"):
        for F, ldb in ((602, 608), (200, 200), (40, 40)):
            Bh = t(synth.dense(700, F, seed=F, ld=ldb)).to(torch.bfloat16)
            ws = es.es_spmm_workspace(300, 700, len(colind), F, ldb, 64, True, device=dev)
            es.es_spmm_run_ex(rp, ci, va, Bh, 64, 2, 5, 1, F=F, workspace=ws)
            dC = t(synth.dense(300, F, seed=3, ld=ldb))
            es.es_spmm_backward_ex(rp, ci, va, dC, 700, 64, 2, 5, 1, F=F, workspace=ws, reuse_sampled=True)
            torch.cuda.synchronize()
            print("ok slab bf16 + backward", F, ldb, flush=True)
    es.es_spmm_sample(rp, ci, va, 40, 2, 9)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    es.es_spmm_run_host(pin(rowptr), pin(colind), pin(val), pin(synth.dense(700, 602, 1, ld=604)), 64, 2, 0,
                        1, F=602)
    torch.cuda.synchronize()
    print("sanitize calls done")


if __name__ == "__main__":
    main()
