"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north_star):
  * sampled edge sets / positions / counts: bit-exact (es_spmm_sample vs oracle.sample);
  * fp32 values: |g - o| <= max(1e-5 |o|, 1e-6) with non-negative inputs (val in [0.5,1.5)
    or 1, B in [0,1)); signed B uses |g - o| <= 1e-5 * sum|val*B| + 1e-6 (cancellation).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_10716_b200 as es  # noqa: E402
from paper_2104_10716_b200 import ES_BUCKET, ES_FASTRAND, ES_REDUCE_MEAN, ES_REDUCE_SUM  # noqa: E402

DEV = "cuda:0"
STRATS = [ES_BUCKET, ES_FASTRAND]


def rel_ok(g, o, rtol=1e-5, atol=1e-6):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    err = np.abs(g - o)
    tol = np.maximum(rtol * np.abs(o), atol)
    bad = err > tol
    if bad.any():
        idx = np.argwhere(bad)[:5]
        return False, f"{bad.sum()} bad, e.g. {[(tuple(i), g[tuple(i)], o[tuple(i)]) for i in idx]}"
    return True, f"max rel {np.max(err / np.maximum(np.abs(o), 1e-30)):.2e}"


def to_dev(rowptr, colind, val):
    return (torch.from_numpy(np.ascontiguousarray(rowptr)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(colind)).to(DEV),
            None if val is None else torch.from_numpy(np.ascontiguousarray(val)).to(DEV))


SLAB_KERNELS = (es.ES_KERNEL_SLAB, es.ES_KERNEL_SLAB_SMEM, es.ES_KERNEL_SLAB_LDG, es.ES_KERNEL_SLAB_TMA,
                es.ES_KERNEL_SLAB_STREAM)
FORCED_RUNS = {"forced": 0, "fallback": 0}


def slab_forced():
    return es._OVERRIDE["kernel"] in SLAB_KERNELS


def run_any(rp, ci, v, Bd, s, strat, seed, reduce, F, C=None):
    """es_spmm_run, or -- under a forced slab kernel -- es_spmm_run_ex with a workspace (the
    feature-sliced path).  A forced family the layout cannot run (ES_ERR_UNSUPPORTED: e.g. the
    slab path at F <= 16, 256-bit gathers on a 16-B row pitch) runs the library's plan instead;
    FORCED_RUNS counts both so a test can check that the forced kernel really ran."""
    try:
        if slab_forced():
            n = rp.numel() - 1
            ws = es.es_spmm_workspace(n, Bd.shape[0], ci.numel(), F, Bd.shape[1], s, v is not None, device=DEV)
            if ws is None:
                raise es.EsError("es_spmm_run_ex failed: ES_ERR_UNSUPPORTED (no slab workspace)")
            out = es.es_spmm_run_ex(rp, ci, v, Bd, s, strat, seed, reduce, F=F, C=C, workspace=ws)
            assert es.es_spmm_workspace_status(ws) == es.ES_WS_OK
        else:
            out = es.es_spmm_run(rp, ci, v, Bd, s, strat, seed, reduce, F=F, C=C)
        FORCED_RUNS["forced"] += 1
        return out
    except es.EsError as exc:
        if "UNSUPPORTED" not in str(exc) or not es.overridden():
            raise
        FORCED_RUNS["fallback"] += 1
        with es.kernel_override("auto"):
            return es.es_spmm_run(rp, ci, v, Bd, s, strat, seed, reduce, F=F, C=C)


def run_gpu(rowptr, colind, val, B, s, strat, seed=0, reduce=ES_REDUCE_SUM, F=None, ldc=None):
    rp, ci, v = to_dev(rowptr, colind, val)
    Bd = torch.from_numpy(np.ascontiguousarray(B)).to(DEV)
    F = B.shape[1] if F is None else F
    n = len(rowptr) - 1
    C = None
    if ldc is not None:
        C = torch.full((n, ldc), -7.0, dtype=torch.float32, device=DEV)
    out = run_any(rp, ci, v, Bd, s, strat, seed, reduce, F, C)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.fixture(scope="module")
def ragged():
    # several tiles of rows, a ragged tail, empty rows, FastRand duplicate degrees
    return synth.random_csr(1237, 3001, seed=17, max_deg=300,
                            special=(577, 1154, 1731, 578, 576, 2000, 1))


# ------------------------------------------------------------------ sampler: bit-exact
@pytest.mark.parametrize("strat", STRATS)
@pytest.mark.parametrize("seed", [0, 7, 2**63 + 5])
@pytest.mark.parametrize("s", [1, 3, 32, 256, 5000])
def test_sample_bit_exact(ragged, strat, seed, s):
    rowptr, colind, val = ragged
    rp, ci, v = to_dev(rowptr, colind, val)
    srp, sc, sv, spos = es.es_spmm_sample(rp, ci, v, s, strat, seed)
    orp, oc, ov, opos = oracle.sample(rowptr, colind, val, s, strat, seed)
    assert np.array_equal(srp.cpu().numpy(), orp)
    assert np.array_equal(sc.cpu().numpy(), oc)
    assert np.array_equal(sv.cpu().numpy().view(np.uint32), ov.view(np.uint32))
    assert np.array_equal(spos.cpu().numpy(), opos)


def test_sample_row_base_and_null_val(ragged):
    rowptr, colind, _ = ragged
    a, b = 100, 900
    rp = torch.from_numpy(rowptr[a:b + 1].copy()).to(DEV)
    ci = torch.from_numpy(colind).to(DEV)
    srp, sc, sv, spos = es.es_spmm_sample(rp, ci, None, 40, ES_FASTRAND, seed=5, row_base=a)
    orp, oc, ov, opos = oracle.sample(rowptr[a:b + 1], colind, None, 40, oracle.FASTRAND, 5, row_base=a)
    assert np.array_equal(srp.cpu().numpy(), orp)
    assert np.array_equal(sc.cpu().numpy(), oc)
    assert np.all(sv.cpu().numpy() == 1.0)
    assert np.array_equal(spos.cpu().numpy(), opos)


# ------------------------------------------------------------------ fused SpMM values
FS = [(1, 1), (3, 3), (3, 4), (7, 8), (16, 16), (17, 17), (32, 32), (64, 64), (100, 100),
      (128, 128), (129, 132), (256, 256), (602, 602), (602, 604), (1000, 1000), (1100, 1104)]


KERNEL_PARAMS = {                       # name -> (kernel family, tune: stages, width, cta_warps, variant)
    "auto": ("auto", ()), "warp": ("warp", ()), "tma": ("tma", ()), "cpasync": ("cpasync", ()),
    "halfwarp": ("halfwarp", ()), "slab": ("slab", ()), "slab16": ("slab_smem", (0, 16)),
    "slab_ldg": ("slab_ldg", ()), "slab_tma": ("slab_tma", ()), "slab_stream": ("slab_stream", (0, 0, 0, 1024)),
    "rowstream": ("rowstream", ()), "grouped": ("grouped", ()), "grouped8": ("grouped", (8,)),
    "grouped_ring": ("grouped", (4, 0, 0, 1)), "segstream": ("segstream", ()),
    "segstream32": ("segstream", (6, 32)),
}


@pytest.fixture(params=list(KERNEL_PARAMS))
def kernel(request):
    """Run a test under the automatic plan and with each kernel family forced where it applies
    (es_spmm_options_t.kernel): LDG warp-per-row, TMA ring, cp.async ring (one / two slots per
    step), and the feature-sliced path with each slab kernel (shared-memory ring with 8 and 16
    lanes per slot, register-direct 256-bit gathers, TMA gather4)."""
    fam, tune = KERNEL_PARAMS[request.param]
    with es.kernel_override(fam, *tune):
        yield request.param


@pytest.mark.parametrize("F,ldb", FS)
@pytest.mark.parametrize("strat", STRATS)
def test_spmm_parity_feature_widths(ragged, F, ldb, strat, kernel):
    rowptr, colind, val = ragged
    B = synth.dense(3001, F, seed=F, ld=ldb)
    for s, seed, reduce in [(32, 0, ES_REDUCE_SUM), (256, 9, ES_REDUCE_MEAN), (3000, 0, ES_REDUCE_SUM)]:
        g = run_gpu(rowptr, colind, val, B, s, strat, seed, reduce, F=F)
        o = oracle.spmm(rowptr, colind, val, B, s, strat, seed=seed, reduce=reduce, F=F)
        ok, msg = rel_ok(g, o)
        assert ok, (F, ldb, s, seed, reduce, msg)


@pytest.mark.parametrize("strat", STRATS)
@pytest.mark.parametrize("s", [1, 2, 5, 31, 33, 64, 200, 577, 1200, 100000])
def test_spmm_parity_s_sweep(ragged, strat, s, kernel):
    rowptr, colind, val = ragged
    B = synth.dense(3001, 128, seed=3)
    for reduce in (ES_REDUCE_SUM, ES_REDUCE_MEAN):
        g = run_gpu(rowptr, colind, val, B, s, strat, 11, reduce)
        o = oracle.spmm(rowptr, colind, val, B, s, strat, seed=11, reduce=reduce)
        ok, msg = rel_ok(g, o)
        assert ok, (s, reduce, msg)


def test_ones_give_exact_counts(ragged, kernel):
    """B == 1, val NULL, SUM: C = k_i exactly, FastRand duplicates included."""
    rowptr, colind, _ = ragged
    d = np.diff(rowptr)
    for F, ldb in ((16, 16), (128, 128), (602, 602), (602, 604)):
        B = np.ones((3001, ldb), np.float32)
        for s in (1, 64, 700):
            for strat in STRATS:
                g = run_gpu(rowptr, colind, None, B, s, strat, seed=3, F=F)
                assert np.array_equal(g, np.repeat(np.minimum(d, s)[:, None], F, 1).astype(np.float32))
                gm = run_gpu(rowptr, colind, None, B, s, strat, seed=3, reduce=ES_REDUCE_MEAN, F=F)
                assert np.array_equal(gm, np.repeat((d > 0)[:, None], F, 1).astype(np.float32))


@pytest.mark.parametrize("F", [65, 100, 128])
@pytest.mark.parametrize("U,ring", [(2, 0), (4, 0), (8, 0), (4, 1), (8, 1)])
def test_grouped_bitwise_warp(ragged, F, U, ring):
    """The degree-sorted half-warp kernel (spmm_grouped) sums each row in slot order with
    32-slot-chunk partials, exactly as the LDG warp-per-row kernel does: bitwise, whatever the
    sort put in each half-warp or how many slots are in flight."""
    rowptr, colind, val = ragged
    B = synth.dense(3001, F, seed=F, ld=(F + 3) // 4 * 4)
    for s, strat, red in ((16, ES_FASTRAND, ES_REDUCE_MEAN), (64, ES_BUCKET, ES_REDUCE_SUM),
                          (700, ES_FASTRAND, ES_REDUCE_MEAN), (1, ES_FASTRAND, ES_REDUCE_SUM)):
        with es.kernel_override("warp"):
            a = run_gpu(rowptr, colind, val, B, s, strat, 5, red, F=F)
        with es.kernel_override("grouped", U, 0, 0, ring):
            b = run_gpu(rowptr, colind, val, B, s, strat, 5, red, F=F)
        assert np.array_equal(a, b), (F, s, strat, ring)


@pytest.mark.parametrize("F", [65, 100, 128])
@pytest.mark.parametrize("ctaw", [2, 4])
@pytest.mark.parametrize("rows,minb", [(8, 6), (16, 6), (32, 6), (4, 7), (8, 7), (16, 7), (32, 7), (8, 8), (16, 8), (32, 8)])
def test_segstream_bitwise_warp(ragged, F, rows, minb, ctaw):
    """The segmented register stream (R rows per warp as one slot stream, row / chunk events from
    lane-parallel ballots) sums each row in slot order with 32-slot chunk partials from the row's
    first slot -- the LDG warp-per-row kernel's order: bitwise, for every rows-per-warp and
    register cap, across row ends inside and between the 4-slot groups and chunks."""
    rowptr, colind, val = ragged
    B = synth.dense(3001, F, seed=F, ld=(F + 3) // 4 * 4)
    for s, strat, red, v in ((16, ES_FASTRAND, ES_REDUCE_MEAN, val), (64, ES_BUCKET, ES_REDUCE_SUM, val),
                             (700, ES_FASTRAND, ES_REDUCE_MEAN, None), (1, ES_FASTRAND, ES_REDUCE_SUM, val),
                             (33, ES_FASTRAND, ES_REDUCE_SUM, None)):
        with es.kernel_override("warp"):
            a = run_gpu(rowptr, colind, v, B, s, strat, 5, red, F=F)
        with es.kernel_override("segstream", minb, rows, ctaw):
            b = run_gpu(rowptr, colind, v, B, s, strat, 5, red, F=F)
        assert np.array_equal(a, b), (F, rows, minb, s, strat)
    # Arxiv-like short rows: most rows 0-5 slots, so several rows end inside one 4-slot group
    rp2, ci2, v2 = synth.random_csr(2011, 3001, seed=23, max_deg=6, special=(40, 33, 64))
    for s, strat in ((64, ES_FASTRAND), (2, ES_BUCKET)):
        with es.kernel_override("warp"):
            a = run_gpu(rp2, ci2, v2, B, s, strat, 9, ES_REDUCE_MEAN, F=F)
        with es.kernel_override("segstream", minb, rows, ctaw):
            b = run_gpu(rp2, ci2, v2, B, s, strat, 9, ES_REDUCE_MEAN, F=F)
        assert np.array_equal(a, b), (F, rows, minb, s, strat, "short rows")


@pytest.mark.parametrize("F", [65, 100, 128])
@pytest.mark.parametrize("rows", [8, 16, 32])
def test_rowstream_bitwise_cpasync(ragged, F, rows):
    """The row stream (several rows per warp as one slot stream) sums each row exactly as the
    one-slot cp.async ring does (32-slot chunk partials from the row's first slot): bitwise."""
    rowptr, colind, val = ragged
    B = synth.dense(3001, F, seed=F, ld=(F + 3) // 4 * 4)
    for s, strat in ((16, ES_FASTRAND), (64, ES_BUCKET), (700, ES_FASTRAND)):
        with es.kernel_override("cpasync"):
            a = run_gpu(rowptr, colind, val, B, s, strat, 5, ES_REDUCE_MEAN, F=F)
        with es.kernel_override("rowstream", 0, rows):
            b = run_gpu(rowptr, colind, val, B, s, strat, 5, ES_REDUCE_MEAN, F=F)
        assert np.array_equal(a, b), (F, rows, s)


def test_s1_bitwise_single_product(ragged):
    rowptr, colind, val = ragged
    B = synth.dense(3001, 40, seed=1)
    for strat in STRATS:
        g = run_gpu(rowptr, colind, val, B, 1, strat)
        o = oracle.spmm(rowptr, colind, val, B, 1, strat)
        assert np.array_equal(g, o)


def test_exact_spmm_vs_cusparse(ragged):
    """s >= max degree = exact SpMM; compare with torch.sparse (cuSPARSE) as a library check."""
    rowptr, colind, val = ragged
    B = synth.dense(3001, 64, seed=2)
    s = int(np.diff(rowptr).max())
    rp, ci, v = to_dev(rowptr, colind, val)
    torch.cuda.synchronize()
    A = torch.sparse_csr_tensor(rp, ci.to(torch.int64), v, size=(len(rowptr) - 1, 3001))
    ref = (A @ torch.from_numpy(B).to(DEV)).cpu().numpy()
    g = run_gpu(rowptr, colind, val, B, s, ES_BUCKET)
    assert np.allclose(g, ref, rtol=2e-5, atol=1e-5)


def test_signed_inputs_condition_aware(ragged):
    rowptr, colind, val = ragged
    rng = np.random.default_rng(4)
    B = (rng.random((3001, 96), dtype=np.float32) * 2 - 1).astype(np.float32)
    sval = (val * np.where(rng.random(len(val)) < 0.5, -1, 1)).astype(np.float32)
    for strat in STRATS:
        g = run_gpu(rowptr, colind, sval, B, 128, strat, 5)
        o = oracle.spmm(rowptr, colind, sval, B, 128, strat, seed=5)
        mag = oracle.spmm(rowptr, colind, np.abs(sval), np.abs(B), 128, strat, seed=5)
        assert np.all(np.abs(g.astype(np.float64) - o) <= 1e-5 * mag + 1e-6)


def test_ldc_padding_untouched_and_misaligned_b(ragged):
    rowptr, colind, val = ragged
    B = synth.dense(3001, 130, seed=5)
    o = oracle.spmm(rowptr, colind, val, B, 48, ES_FASTRAND, seed=1, F=130)
    g = run_gpu(rowptr, colind, val, B, 48, ES_FASTRAND, seed=1, F=130, ldc=133)
    assert np.all(g[:, 130:] == -7.0)
    assert rel_ok(g[:, :130], o)[0]
    # B starting at a 4-byte offset -> scalar gather path
    rp, ci, v = to_dev(rowptr, colind, val)
    big = torch.from_numpy(np.concatenate([np.zeros(1, np.float32), B.ravel()])).to(DEV)
    Bmis = big[1:].view(3001, 130)
    assert "vec1" in es.es_spmm_plan(130, 130, 130, Bmis, None) or "vec2" in es.es_spmm_plan(130, 130, 130, Bmis, None)
    C = es.es_spmm_run(rp, ci, v, Bmis, 48, ES_FASTRAND, 1)
    assert rel_ok(C.cpu().numpy(), o)[0]


def test_row_slices_bitwise_equal_full(ragged, kernel):
    """The multi-GPU invariant: row blocks on a CSR slice == rows of the full launch, bitwise."""
    rowptr, colind, val = ragged
    B = synth.dense(3001, 602, seed=8, ld=604)
    Bd = torch.from_numpy(B).to(DEV)
    rp, ci, v = to_dev(rowptr, colind, val)
    full = run_any(rp, ci, v, Bd, 256, ES_FASTRAND, 99, ES_REDUCE_MEAN, 602).cpu().numpy()
    bounds = es.es_partition_rows(rowptr, 256, 602, 3)
    for a, b in zip(bounds[:-1], bounds[1:]):
        e0, e1 = rowptr[a], rowptr[b]
        rps = torch.from_numpy(rowptr[a:b + 1].copy()).to(DEV)
        cis = torch.from_numpy(colind[e0:e1].copy()).to(DEV)
        vs = torch.from_numpy(val[e0:e1].copy()).to(DEV)
        if slab_forced() and es._OVERRIDE["kernel"] != es.ES_KERNEL_SLAB_LDG:      # (604: no 32-B pitch)
            ws = es.es_spmm_workspace(int(b - a), 3001, int(e1 - e0), 602, 604, 256, True, device=DEV)
            part = es.es_spmm_run_ex(rps, cis, vs, Bd, 256, ES_FASTRAND, 99, ES_REDUCE_MEAN, F=602,
                                     row_begin=int(a), row_end=int(b), n_rows=len(rowptr) - 1,
                                     nnz_base=int(e0), workspace=ws, nnz=int(e1 - e0)).cpu().numpy()
        else:
            part = es.es_spmm_run_rows(len(rowptr) - 1, rps, int(e0), cis, vs, Bd, 256, ES_FASTRAND, 99,
                                       ES_REDUCE_MEAN, int(a), int(b), F=602).cpu().numpy()
        assert np.array_equal(part, full[a:b])


def test_host_api_matches_device_api(ragged):
    rowptr, colind, val = ragged
    B = synth.dense(3001, 602, seed=8, ld=604)
    pin = lambda a: torch.from_numpy(a).pin_memory()
    Ch = es.es_spmm_run_host(pin(rowptr), pin(colind), pin(val), pin(B), 200, ES_FASTRAND, 4,
                             ES_REDUCE_MEAN, F=602)
    rp, ci, v = to_dev(rowptr, colind, val)
    Cd = es.es_spmm_run(rp, ci, v, torch.from_numpy(B).to(DEV), 200, ES_FASTRAND, 4, ES_REDUCE_MEAN,
                        F=602).cpu().numpy()
    assert np.array_equal(Ch.numpy(), Cd)


def test_empty_inputs():
    B = torch.zeros((4, 8), device=DEV)
    rp = torch.zeros(1, dtype=torch.int64, device=DEV)
    ci = torch.zeros(0, dtype=torch.int32, device=DEV)
    C = es.es_spmm_run(rp, ci, None, B, 4, ES_FASTRAND)
    assert C.shape == (0, 8)
    rp = torch.zeros(6, dtype=torch.int64, device=DEV)
    C = es.es_spmm_run(rp, ci, None, B, 4, ES_FASTRAND, reduce=ES_REDUCE_MEAN)
    torch.cuda.synchronize()
    assert torch.all(C == 0)
    srp, sc, sv, spos = es.es_spmm_sample(rp, ci, None, 3, ES_BUCKET)
    assert srp.cpu().tolist() == [0] * 6 and sc.numel() == 0


def test_launch_counter_moves(ragged):
    rowptr, colind, val = ragged
    n0 = es.es_launch_count()
    run_gpu(rowptr, colind, val, synth.dense(3001, 16, seed=1), 8, ES_FASTRAND)
    assert es.es_launch_count() == n0 + 1


# ------------------------------------------------------------------ full-size configs
_ORACLE_CACHE = {}


def _oracle_full(name, F, s, strat, seed, reduce, rowptr, colind, val, B, rows):
    """The oracle's C for a full-size config (every row unless `rows`), cached across the kernel
    parametrisations (the values do not depend on B's row padding)."""
    key = (name, F, s, strat, seed, reduce, None if rows is None else len(rows))
    if key not in _ORACLE_CACHE:
        if len(_ORACLE_CACHE) >= 2:
            _ORACLE_CACHE.pop(next(iter(_ORACLE_CACHE)))
        _ORACLE_CACHE[key] = oracle.spmm(rowptr, colind, val, B, s, strat, seed=seed, reduce=reduce, F=F,
                                         rows=rows)
    return _ORACLE_CACHE[key]


def _full(name, F, ldb, s, strat, seed, reduce, sample=None):
    """A full-size config in the bench launch configuration, checked against the oracle on EVERY
    row (sample=None), or -- for the 1B-edge graph -- on a seeded 1/sample row sample plus the
    1,000 highest-degree rows."""
    rowptr, colind = synth.graph(name)
    n = len(rowptr) - 1
    _, seed_b = synth.seeds(name)
    B = synth.dense(n, F, seed_b, ld=ldb)
    val = np.ones(len(colind), np.float32)
    rp, ci, v = to_dev(rowptr, colind, val)
    Bd = torch.from_numpy(B).to(DEV)
    C = run_any(rp, ci, v, Bd, s, strat, seed, reduce, F)
    torch.cuda.synchronize()
    d = np.diff(rowptr)
    rng = np.random.default_rng(0)
    if sample is None:
        rows = None
        g = C[:, :F].cpu().numpy()
    else:
        rows = np.unique(np.concatenate([rng.choice(n, n // sample, replace=False),
                                         np.argsort(-d, kind="stable")[:1000], [0, n - 1]])).astype(np.int64)
        g = C[torch.from_numpy(rows).to(DEV)][:, :F].cpu().numpy()
    o = _oracle_full(name, F, s, strat, seed, reduce, rowptr, colind, val, B, rows)
    ok, msg = rel_ok(g, o)
    assert ok, (name, msg)
    # sampler at full size: k_i of every row, and the bit-exact slot positions / columns of a
    # row sample against the brute-force Eq. 2 positions
    srp, sc, _, spos = es.es_spmm_sample(rp, ci, v, s, strat, seed, want_pos=True)
    srp = srp.cpu().numpy()
    assert np.array_equal(np.diff(srp), np.minimum(d, s))
    check = np.unique(np.concatenate([rng.choice(n, 200, replace=False), np.argsort(-d, kind="stable")[:200]]))
    for r in check:
        a, b = int(srp[r]), int(srp[r + 1])
        want = oracle.brute.positions(strat, int(d[r]), s, seed, int(r))
        assert spos[a:b].cpu().tolist() == want
        assert np.array_equal(sc[a:b].cpu().numpy(), colind[rowptr[r] + np.asarray(want, np.int64)])
    return msg


@pytest.mark.parametrize("strat", STRATS)
def test_full_pubmed(strat):
    rowptr, colind = synth.graph("pubmed")
    n = len(rowptr) - 1
    B = synth.dense(n, 16, synth.seeds("pubmed")[1])
    g = run_gpu(rowptr, colind, None, B, 32, strat, 0, ES_REDUCE_MEAN)
    o = oracle.spmm(rowptr, colind, None, B, 32, strat, reduce=oracle.MEAN)
    assert rel_ok(g, o)[0]


@pytest.mark.parametrize("s", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("strat", STRATS)
def test_full_arxiv(s, strat):
    _full("arxiv", 128, 128, s, strat, 0, ES_REDUCE_SUM)


@pytest.mark.parametrize("path", ["fused", "slab"])
def test_full_proteins(path):
    """Config 3 at full size; bench.py takes the slab path here (long rows), so both are checked."""
    with es.kernel_override(path):
        _full("proteins", 128, 128, 256, ES_FASTRAND, 0, ES_REDUCE_SUM)


@pytest.mark.parametrize("F,ldb", [(602, 608), (602, 604), (128, 128)])   # 608 = bench.py layout
@pytest.mark.parametrize("strat", STRATS)
def test_full_reddit(F, ldb, strat, kernel):
    _full("reddit", F, ldb, 256, strat, 0, ES_REDUCE_MEAN)


@pytest.mark.slow
@pytest.mark.parametrize("strat", [ES_FASTRAND])
def test_full_scaled(strat):
    """Config 5: 10M nodes, 1.0B edges, F=256, s=128 (bench launch configuration, 1 GPU)."""
    _full("scaled", 256, 256, 128, strat, 0, ES_REDUCE_SUM, sample=64)


def test_hand_golden_exact(golden, kernel):
    """The hand-checkable worked example (tests/golden/worked_examples.json 'hand'): small
    integers, so every kernel family must reproduce it exactly."""
    g = golden["hand"]
    rowptr = np.array(g["rowptr"], np.int64)
    colind = np.array(g["colind"], np.int32)
    for F in (2, 130, 602):          # subwarp / warp-or-cpasync / tma paths; extra columns = 0
        B = np.zeros((g["n_cols"], F if F != 602 else 604), np.float32)
        B[:, 0] = np.arange(1, g["n_cols"] + 1)
        B[:, 1] = 10 * np.arange(1, g["n_cols"] + 1)
        for c in g["cases"]:
            strat = ES_BUCKET if c["strategy"] == "bucket" else ES_FASTRAND
            red = ES_REDUCE_SUM if c["reduce"] == "sum" else ES_REDUCE_MEAN
            out = run_gpu(rowptr, colind, None, B, c["s"], strat, 0, red, F=F)
            assert np.array_equal(out[:, :2], np.array(c["C"], np.float32)), (F, c)
            assert np.all(out[:, 2:] == 0)
