"""Edge cases of the CUDA path against the oracle: stored (unsorted) column order, duplicate
columns, the 64-bit FastRand position path, huge s, hub rows, empty B."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_10716_b200 as es  # noqa: E402

DEV = "cuda:0"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def close(g, o):
    err = np.abs(np.asarray(g, np.float64) - o)
    return bool(np.all(err <= np.maximum(1e-5 * np.abs(o), 1e-6)))


@pytest.mark.parametrize("F,ld", [(16, 16), (128, 128), (602, 604)])
def test_unsorted_rows_follow_stored_order(F, ld):
    """Reading R4: Bucket keeps the first k STORED entries; nothing assumes sorted columns."""
    rowptr, colind, val = synth.random_csr(700, 1500, seed=40, max_deg=200)
    rng = np.random.default_rng(1)
    ci = colind.copy()
    for i in range(700):
        a, b = rowptr[i], rowptr[i + 1]
        ci[a:b] = rng.permutation(ci[a:b])
    B = synth.dense(1500, F, seed=2, ld=ld)
    for strat in (1, 2):
        g = es.es_spmm_run(t(rowptr), t(ci), t(val), t(B), 24, strat, 0, 1, F=F).cpu().numpy()
        o = oracle.spmm(rowptr, ci, val, B, 24, strat, reduce=1, F=F)
        assert close(g, o)
        g_sorted = es.es_spmm_run(t(rowptr), t(colind), t(val), t(B), 24, 1, 0, 1, F=F).cpu().numpy()
        if strat == 1:
            assert not np.array_equal(g, g_sorted)      # the order matters for Bucket


def test_duplicate_columns_in_a_row():
    rowptr = np.array([0, 6, 10], np.int64)
    colind = np.array([3, 3, 3, 1, 3, 0, 2, 2, 2, 2], np.int32)
    val = np.linspace(0.5, 1.4, 10).astype(np.float32)
    B = synth.dense(4, 130, seed=5, ld=132)
    for strat in (1, 2):
        for s in (1, 3, 6, 100):
            g = es.es_spmm_run(t(rowptr), t(colind), t(val), t(B), s, strat, 9, 0, F=130).cpu().numpy()
            o = oracle.spmm(rowptr, colind, val, B, s, strat, seed=9, F=130)
            assert close(g, o)


def test_64bit_fastrand_position_path():
    """A row with k = 7.5M slots: (k-1)*577 >= 2^32, so positions take the 64-bit path."""
    d = 7_500_000
    rowptr = np.array([0, d], np.int64)
    colind = (np.arange(d, dtype=np.int64) % 1000).astype(np.int32)
    srp, sc, _, spos = es.es_spmm_sample(t(rowptr), t(colind), None, d, 2, seed=3)
    orp, oc, _, opos = oracle.sample(rowptr, colind, None, d, 2, seed=3)
    assert np.array_equal(spos.cpu().numpy(), opos)
    assert np.array_equal(sc.cpu().numpy(), oc)
    B = np.ones((1000, 4), np.float32)
    g = es.es_spmm_run(t(rowptr), t(colind), None, t(B), d, 2, 3, 0).cpu().numpy()
    assert np.array_equal(g, np.full((1, 4), d, np.float32))


def test_huge_s_and_hub_rows():
    rng = np.random.default_rng(7)
    degs = np.array([0, 1, 200_000, 577 * 40, 5, 150_000], np.int64)
    rowptr = np.concatenate([[0], np.cumsum(degs)])
    colind = rng.integers(0, 300_000, int(rowptr[-1])).astype(np.int32)
    val = rng.random(int(rowptr[-1]), dtype=np.float32) + 0.5
    B = synth.dense(300_000, 128, seed=1)
    for s in (2**31 - 1, 5000):
        for strat in (1, 2):
            g = es.es_spmm_run(t(rowptr), t(colind), t(val), t(B), s, strat, 11, 1).cpu().numpy()
            o = oracle.spmm(rowptr, colind, val, B, s, strat, seed=11, reduce=1)
            assert close(g, o), (s, strat)


def test_no_columns_and_no_rows():
    rowptr = np.zeros(5, np.int64)
    colind = np.zeros(0, np.int32)
    B = torch.zeros((0, 8), device=DEV)
    C = es.es_spmm_run(t(rowptr), t(colind), None, B, 4, 2, 0, 1)
    torch.cuda.synchronize()
    assert C.shape == (4, 8) and bool(torch.all(C == 0))
