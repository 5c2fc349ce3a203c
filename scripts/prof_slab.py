#!/usr/bin/env python3
"""ncu driver (tuning evidence only): the slab path on the Reddit-shaped graph, F=602.
Runs the slab call 3 times (L2 flushed before each); profile with -k regex:spmm_slab -s 20 -c 1."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402
from bench import ldb_for  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 602
ldb = ldb_for(F)
dev = torch.device("cuda:0")
rowptr, colind = synth.graph("reddit")
n = len(rowptr) - 1
B = torch.from_numpy(synth.dense(n, F, synth.seeds("reddit")[1], ld=ldb)).to(dev)
rp = torch.from_numpy(rowptr).to(dev)
ci = torch.from_numpy(colind).to(dev)
va = torch.ones(len(colind), dtype=torch.float32, device=dev)
C = torch.zeros((n, ldb), dtype=torch.float32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
os.environ.setdefault("ES_SPMM_SLAB", "1")
ws = es.es_spmm_workspace(n, n, len(colind), F, ldb, 256, True, device=dev)
for i in range(3):
    flush.zero_()
    es.es_spmm_run_ex(rp, ci, va, B, 256, 2, 0, 1, F=F, C=C, workspace=ws)
torch.cuda.synchronize()
print("ok")
