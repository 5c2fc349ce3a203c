"""Downstream check (north_star): 2-layer GCN / GraphSage-mean logits with seeded random
weights, GPU path (sampled SpMM kernels + fp32 GEMM, TF32 off) vs the oracle (fp64 GEMM +
C oracle SpMM): argmax agreement and logits error."""
import numpy as np
import pytest

import oracle
import oracle.gnn as ognn
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2104_10716_b200 import gnn  # noqa: E402


@pytest.mark.parametrize("model", ["gcn", "sage"])
@pytest.mark.parametrize("strategy", [1, 2])
def test_small_graph_argmax_agreement(model, strategy):
    rowptr, colind, val = synth.random_csr(3000, 3000, seed=4, max_deg=200, special=(577,))
    X = synth.dense(3000, 50, seed=6, ld=52)
    layers = gnn.init_weights(model, [50, 32, 7], seed=1)
    dev = "cuda:0"
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    g = gnn.forward(model, t(rowptr), t(colind), t(val), t(X), layers, 16, strategy, seed=3).cpu().numpy()
    o = ognn.forward(model, rowptr, colind, val, X, layers, 16, strategy, seed=3)
    agree = np.mean(gnn.argmax_lowest(g) == gnn.argmax_lowest(o))
    assert agree >= 0.999, agree
    assert np.max(np.abs(g - o)) <= 1e-4 * max(1.0, np.max(np.abs(o)))
