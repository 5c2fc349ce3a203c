#!/usr/bin/env python3
"""One launch each of: our fused kernel (Reddit F=128, s=256 FastRand) and cuSPARSE on the
pre-sampled CSR, for an ncu --set full comparison."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa
import paper_2104_10716_b200 as es  # noqa

name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
s = int(sys.argv[2]) if len(sys.argv) > 2 else 256
dev = torch.device("cuda:0")
rowptr, colind = synth.graph(name)
n = len(rowptr) - 1
B = torch.from_numpy(synth.dense(n, 128, 3)).to(dev)
rp, ci = torch.from_numpy(rowptr).to(dev), torch.from_numpy(colind).to(dev)
va = torch.ones(len(colind), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
srp, sc, sv, _ = es.es_spmm_sample(rp, ci, va, s, 2, 0, want_pos=False)
As = torch.sparse_csr_tensor(srp.to(torch.int32), sc, sv, size=(n, n))
for _ in range(3):
    flush.zero_(); es.es_spmm_run(rp, ci, va, B, s, 2, 0, 0)
    flush.zero_(); As @ B
torch.cuda.synchronize()
