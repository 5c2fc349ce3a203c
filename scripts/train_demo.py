#!/usr/bin/env python3
"""Training variant demo (NEXT-2): full-graph GraphSage-mean training where every iteration
draws a NEW sampled subset (seed = iteration; reading R6) -- the DropEdge-style dynamic
sampling the paper leaves to future work (§6.2) -- through the autograd op
(forward es_spmm_run, backward es_spmm_backward).

Task (synthetic, no datasets here): labels = argmax of a random "teacher" GraphSage layer on
the exact graph; the student trains on sampled aggregations.  Reports loss / accuracy on the
exact graph and per-iteration time vs training on the exact graph (s >= max degree).
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2104_10716_b200 import ES_FASTRAND, ES_REDUCE_MEAN, es_spmm_run  # noqa: E402
from paper_2104_10716_b200.autograd import sampled_spmm  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 60
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph(name)
    n = len(rowptr) - 1
    dmax = int(np.diff(rowptr).max())
    X = torch.from_numpy(synth.dense(n, F, synth.seeds(name)[1])).to(dev)
    X = (X - X.mean(0)) / X.std(0)
    rp, ci = torch.from_numpy(rowptr).to(dev), torch.from_numpy(colind).to(dev)
    n_cls, hid = 16, 128
    g = torch.Generator(device="cpu").manual_seed(0)
    Wt = torch.randn(F, n_cls, generator=g).to(dev)
    with torch.no_grad():                               # teacher on the exact graph
        y = (es_spmm_run(rp, ci, None, X.contiguous(), dmax, ES_FASTRAND, 0, ES_REDUCE_MEAN) @ Wt).argmax(1)

    def run(s, label):
        torch.manual_seed(1)
        lin = torch.nn.ModuleDict({k: torch.nn.Linear(a, b) for k, (a, b) in
                                   {"s1": (F, hid), "n1": (F, hid), "s2": (hid, n_cls), "n2": (hid, n_cls)}.items()}).to(dev)
        opt = torch.optim.Adam(lin.parameters(), lr=0.01)
        log = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for it in range(iters):
            seed = it + 1 if s < dmax else 0               # a new subset every iteration
            agg0 = sampled_spmm(X, rp, ci, None, s, ES_FASTRAND, seed, ES_REDUCE_MEAN)
            h1 = torch.relu(lin["s1"](X) + lin["n1"](agg0))
            agg1 = sampled_spmm(h1, rp, ci, None, s, ES_FASTRAND, seed, ES_REDUCE_MEAN)
            out = lin["s2"](h1) + lin["n2"](agg1)
            loss = torch.nn.functional.cross_entropy(out, y)
            opt.zero_grad()
            loss.backward()
            opt.step()
            if it % 10 == 0 or it == iters - 1:
                log.append((it, round(loss.item(), 4)))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / iters
        with torch.no_grad():                           # evaluate on the exact graph
            agg0 = es_spmm_run(rp, ci, None, X.contiguous(), dmax, ES_FASTRAND, 0, ES_REDUCE_MEAN)
            h1 = torch.relu(lin["s1"](X) + lin["n1"](agg0))
            out = lin["s2"](h1) + lin["n2"](es_spmm_run(rp, ci, None, h1.contiguous(), dmax, ES_FASTRAND, 0,
                                                        ES_REDUCE_MEAN))
            acc = float((out.argmax(1) == y).float().mean())
        print(json.dumps({"graph": name, "F": F, "train": label, "s": s, "iters": iters,
                          "ms_per_iter": round(1e3 * dt, 2), "loss_log": log, "exact_graph_accuracy": round(acc, 4)}),
              flush=True)

    run(dmax, "exact (s >= max degree)")
    for s in (16, 64):
        run(s, f"sampled s={s}, new FastRand subset per iteration")


if __name__ == "__main__":
    main()
