"""NEXT-4 sensitivity variants on the GPU against the oracle: P' override (bit-exact sampled
sets), MEAN by the original degree, bf16 storage of B (oracle fed the same bf16 values, so the
fp32-accumulation bar of 1e-5 still applies)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_10716_b200 as es  # noqa: E402
from _bounds import bound_ok  # noqa: E402

DEV = "cuda:0"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def rel_ok(g, o, rtol=1e-5, atol=1e-6):
    err = np.abs(np.asarray(g, np.float64) - np.asarray(o, np.float64))
    return bool(np.all(err <= np.maximum(rtol * np.abs(o), atol))), float(err.max())


@pytest.fixture(scope="module")
def graph():
    return synth.random_csr(1100, 2300, seed=31, max_deg=300, special=(577, 1009, 2018, 1154, 14))


@pytest.mark.parametrize("prime", [1, 2, 7, 1009])
def test_prime_override(graph, prime):
    rowptr, colind, val = graph
    srp, sc, sv, spos = es.es_spmm_sample_ex(t(rowptr), t(colind), t(val), 40, 2, 5, prime=prime)
    orp, oc, ov, opos = oracle.sample(rowptr, colind, val, 40, 2, 5, prime=prime)
    assert np.array_equal(srp.cpu().numpy(), orp) and np.array_equal(spos.cpu().numpy(), opos)
    assert np.array_equal(sc.cpu().numpy(), oc)
    for F, ld in [(16, 16), (128, 128), (602, 604)]:
        B = synth.dense(2300, F, seed=F, ld=ld)
        g = es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 40, 2, 5, 1, F=F, prime=prime).cpu().numpy()
        o = oracle.spmm(rowptr, colind, val, B, 40, 2, seed=5, reduce=1, F=F, prime=prime)
        assert rel_ok(g, o)[0], (F, prime)
    dC = synth.dense(1100, 24, seed=2)
    dB = es.es_spmm_backward_ex(t(rowptr), t(colind), t(val), t(dC), 2300, 40, 2, 5, 1, prime=prime)
    ok, worst = bound_ok(dB.cpu().numpy(), rowptr, colind, val, dC, 2300, 40, 2, 5, 1, prime=prime)
    assert ok, (prime, worst)


def test_mean_by_degree(graph):
    rowptr, colind, val = graph
    d = np.diff(rowptr)
    for F, ld in [(16, 16), (128, 128), (256, 256), (602, 604)]:
        ones = np.ones((2300, ld), np.float32)
        g = es.es_spmm_run_ex(t(rowptr), t(colind), None, t(ones), 64, 2, 0, 1, F=F, mean_by_degree=True)
        k = np.minimum(d, 64)
        want = np.where(d > 0, k.astype(np.float32) / np.maximum(d, 1).astype(np.float32), 0).astype(np.float32)
        assert np.array_equal(g.cpu().numpy(), np.repeat(want[:, None], F, 1)), F
        B = synth.dense(2300, F, seed=3, ld=ld)
        g = es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 64, 1, 0, 1, F=F, mean_by_degree=True)
        o = oracle.spmm(rowptr, colind, val, B, 64, 1, reduce=1, F=F, mean_by_degree=True)
        assert rel_ok(g.cpu().numpy(), o)[0], F


@pytest.mark.parametrize("F,ld", [(8, 8), (16, 16), (100, 104), (128, 128), (256, 256), (602, 608), (1100, 1104)])
@pytest.mark.parametrize("strat", [1, 2])
@pytest.mark.parametrize("path", ["fused", "slab"])
def test_bf16_storage(graph, F, ld, strat, path):
    rowptr, colind, val = graph
    B32 = synth.dense(2300, F, seed=F + 7, ld=ld)
    Bh = t(B32).to(torch.bfloat16)
    Bq = Bh.float().cpu().numpy()          # the exact values the kernel reads
    ws = None
    if path == "slab":                     # 128-element bf16 slices (+ narrow tails)
        ws = es.es_spmm_workspace(1100, 2300, len(colind), F, ld, 256, True, device=DEV, kernel="slab")
    for s, reduce in [(16, 0), (256, 1)]:
        g = es.es_spmm_run_ex(t(rowptr), t(colind), t(val), Bh, s, strat, 3, reduce, F=F, workspace=ws,
                              kernel="slab" if ws is not None else None).cpu().numpy()
        o = oracle.spmm(rowptr, colind, val, Bq, s, strat, seed=3, reduce=reduce, F=F)
        ok, err = rel_ok(g, o)
        assert ok, (F, s, err)
