"""GPU parity of the backward w.r.t. B (NEXT-2) against the oracle.

The GPU adds contributions with fp32 vector reductions in nondeterministic order, so the bar is
the order-independent bound |g - o| <= (n_c + 2) u sum|terms| (n_c = contributions to that
element, u = 2^-24), computed from the oracle on |val|, |dC|; integer-valued cases are exact."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_10716_b200 as es  # noqa: E402
from paper_2104_10716_b200.autograd import sampled_spmm  # noqa: E402
from _bounds import U, bound_ok  # noqa: E402,F401

DEV = "cuda:0"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.fixture(scope="module")
def graph():
    return synth.random_csr(900, 1100, seed=21, max_deg=250, special=(577, 1154, 1000))


@pytest.mark.parametrize("F,ld", [(1, 1), (16, 16), (41, 41), (128, 128), (602, 604), (602, 602), (1100, 1100)])
@pytest.mark.parametrize("strat", [1, 2])
@pytest.mark.parametrize("reduce", [0, 1])
def test_backward_parity(graph, F, ld, strat, reduce):
    rowptr, colind, val = graph
    dC = synth.dense(900, F, seed=F + 1, ld=ld)
    dB = es.es_spmm_backward(t(rowptr), t(colind), t(val), t(dC), 1100, 64, strat, 9, reduce, F=F, ldb=ld)
    torch.cuda.synchronize()
    g = dB.cpu().numpy()
    ok, worst = bound_ok(g[:, :F], rowptr, colind, val, dC[:, :F], 1100, 64, strat, 9, reduce)
    assert ok, worst
    if ld > F:
        assert np.all(g[:, F:] == 0)          # padding columns never touched


def test_backward_ones_exact(graph):
    rowptr, colind, _ = graph
    for s in (1, 32, 3000):
        dB = es.es_spmm_backward(t(rowptr), t(colind), None, torch.ones((900, 8), device=DEV), 1100, s, 2, 4)
        _, sc, _, _ = oracle.sample(rowptr, colind, None, s, 2, 4)
        hits = np.bincount(sc, minlength=1100).astype(np.float32)
        assert np.array_equal(dB.cpu().numpy(), np.repeat(hits[:, None], 8, 1))


def test_adjoint_identity_gpu(graph):
    rowptr, colind, val = graph
    B = synth.dense(1100, 96, seed=3)
    dC = synth.dense(900, 96, seed=4)
    for reduce in (0, 1):
        C = es.es_spmm_run(t(rowptr), t(colind), t(val), t(B), 50, 2, 7, reduce)
        dB = es.es_spmm_backward(t(rowptr), t(colind), t(val), t(dC), 1100, 50, 2, 7, reduce)
        lhs = float(torch.sum(C.double() * t(dC).double()))
        rhs = float(torch.sum(t(B).double() * dB.double()))
        assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


def test_row_blocks_accumulate_into_one_dB(graph):
    rowptr, colind, val = graph
    dC = synth.dense(900, 64, seed=5)
    full = es.es_spmm_backward(t(rowptr), t(colind), t(val), t(dC), 1100, 40, 2, 3, 1)
    dB = torch.zeros((1100, 64), device=DEV)
    bounds = es.es_partition_rows(rowptr, 40, 64, 3)
    for a, b in zip(bounds[:-1], bounds[1:]):
        e0, e1 = rowptr[a], rowptr[b]
        es.es_spmm_backward(t(rowptr[a:b + 1]), t(colind[e0:e1]), t(val[e0:e1]), t(dC[a:b]), 1100, 40, 2, 3, 1,
                            dB=dB, row_begin=int(a), row_end=int(b), n_rows=900, nnz_base=int(e0))
    assert torch.allclose(dB, full, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("path", ["fused", "slab"])
def test_autograd_gradient(graph, path):
    rowptr, colind, val = graph
    F = 32 if path == "fused" else 136
    B = t(synth.dense(1100, F, seed=8)).requires_grad_(True)
    W = t(synth.dense(900, F, seed=9))
    ws = None
    if path == "slab":                      # forward samples into the workspace, backward reuses it
        ws = es.es_spmm_workspace(900, 1100, len(colind), F, F, 24, True, device=DEV, kernel="slab")
    for seed in (1, 2):                     # a new sampled subset per "iteration"
        with es.kernel_override("slab" if ws is not None else "auto"):
            C = sampled_spmm(B, t(rowptr), t(colind), t(val), 24, 2, seed, 1, workspace=ws)
        loss = (C * W).sum()
        B.grad = None
        loss.backward()
        g = B.grad.cpu().numpy()
        ok, worst = bound_ok(g, rowptr, colind, val, W.cpu().numpy(), 1100, 24, 2, seed, 1)
        assert ok, worst


@pytest.mark.parametrize("F", [1, 40, 128, 602])
@pytest.mark.parametrize("reduce", [0, 1])
def test_deterministic_backward_parity_and_reproducibility(graph, F, reduce):
    rowptr, colind, val = graph
    dC = synth.dense(900, F, seed=F + 3)
    runs = [es.es_spmm_backward_ex(t(rowptr), t(colind), t(val), t(dC), 1100, 64, 2, 9, reduce,
                                   deterministic=True).cpu().numpy() for _ in range(3)]
    assert all(np.array_equal(runs[0].view(np.uint32), r.view(np.uint32)) for r in runs[1:])
    ok, worst = bound_ok(runs[0], rowptr, colind, val, dC, 1100, 64, 2, 9, reduce)
    assert ok, worst
    ones = es.es_spmm_backward_ex(t(rowptr), t(colind), None, torch.ones((900, F), device=DEV), 1100, 64, 2, 9,
                                  deterministic=True).cpu().numpy()
    _, sc, _, _ = oracle.sample(rowptr, colind, None, 64, 2, 9)
    assert np.array_equal(ones, np.repeat(np.bincount(sc, minlength=1100).astype(np.float32)[:, None], F, 1))


@pytest.mark.parametrize("F,ld", [(17, 20), (64, 64), (128, 128), (602, 604), (602, 608)])
@pytest.mark.parametrize("strat", [1, 2])
@pytest.mark.parametrize("reduce", [0, 1])
def test_slab_backward_parity(graph, F, ld, strat, reduce):
    """The feature-sliced backward (a workspace passed): sampling its own slots, and reusing the
    ones a forward call left in the workspace -- same order-independent bound."""
    with es.kernel_override("slab"):
        _slab_backward_parity(graph, F, ld, strat, reduce)


def _slab_backward_parity(graph, F, ld, strat, reduce):
    rowptr, colind, val = graph
    dC = synth.dense(900, F, seed=F + 3, ld=ld)
    B = synth.dense(1100, F, seed=F + 4, ld=ld)
    ws = es.es_spmm_workspace(900, 1100, len(colind), F, ld, 64, True, device=DEV)
    for reuse in (False, True):
        if reuse:                                   # forward samples into the workspace first
            es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 64, strat, 9, reduce, F=F, workspace=ws)
        dB = torch.zeros((1100, ld), dtype=torch.float32, device=DEV)
        es.es_spmm_backward_ex(t(rowptr), t(colind), t(val), t(dC), 1100, 64, strat, 9, reduce, F=F, dB=dB,
                               workspace=ws, reuse_sampled=reuse)
        g = dB.cpu().numpy()
        ok, worst = bound_ok(g[:, :F], rowptr, colind, val, dC[:, :F], 1100, 64, strat, 9, reduce)
        assert ok, (reuse, worst)
        if ld > F:
            assert np.all(g[:, F:] == 0)
