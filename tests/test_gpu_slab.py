"""The feature-sliced ("slab") path of es_spmm_run_ex (es_slab.cu) on the GPU:
parity with the oracle (values within the 1e-5 bar, val NULL, MEAN by degree, the P' option),
the documented per-element order (G = 16 is bitwise spmm_cpasync_hw), row blocks bitwise equal
to the full launch, and the workspace contract."""
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


def rel_ok(g, o, rtol=1e-5, atol=1e-6):
    err = np.abs(np.asarray(g, np.float64) - np.asarray(o, np.float64))
    return bool(np.all(err <= np.maximum(rtol * np.abs(o), atol))), float(err.max())


@pytest.fixture(scope="module")
def graph():
    # several 8-row CTAs, a ragged tail, empty rows, rows past s, FastRand duplicate degrees
    return synth.random_csr(1301, 2300, seed=41, max_deg=400, special=(577, 1154, 1009, 300, 65, 33, 1))


@pytest.fixture(params=["flow", "flow_mp16", "flow_mp8", "flow_w4", "flow_d8", "smem8", "smem16", "ldg", "tma",
                        "stream2", "stream8"])
def lanes(request):
    """Each slab kernel, forced: the flow kernel (the plan's slicing; slices of 16 pieces, of 8;
    4-warp CTAs; an 8-step ring), the per-row shared-memory ring with 8 / 16 lanes per slot, the
    register-direct 256-bit kernel (32-B row pitches; else the plan's), the TMA gather4 kernel,
    the row-pipelined stream (2 / 8 rows per warp)."""
    fam, tune = {"flow": ("slab_flow", ()), "flow_mp16": ("slab_flow", (0, 16)), "flow_mp8": ("slab_flow", (0, 8)),
                 "flow_w4": ("slab_flow", (0, 0, 4)), "flow_d8": ("slab_flow", (8,)),
                 "smem8": ("slab_smem", (0, 8)), "smem16": ("slab_smem", (0, 16)), "ldg": ("slab_ldg", ()),
                 "tma": ("slab_tma", ()), "stream2": ("slab_stream", (0, 0, 0, 512)),
                 "stream8": ("slab_stream", (0, 0, 0, 2048))}[request.param]
    with es.kernel_override(fam, *tune):
        yield request.param


def _unsupported_ok(B):
    """slab_ldg needs a 32-B row pitch: other layouts are ES_ERR_UNSUPPORTED under it."""
    return es._OVERRIDE["kernel"] == es.ES_KERNEL_SLAB_LDG and (B.shape[1] * B.itemsize) % 32 != 0


def flow_launches(F, reuse=False, bf16=False, n_cols=2300):
    """Launches of one flow-path call: count + CUB scan (2) + materialise, then one pass per
    slice of MP 16-B pieces, a remainder of <= 32 - MP (bf16: 24 - MP) pieces merged into the last slice; MP =
    tune width 8 / 16 / 24, else whichever of 16 and 24 needs fewer passes (24 while n_cols x
    384 B <= 96 MB)."""
    npieces = -(-F * (2 if bf16 else 4) // 16)

    def passes(mp):
        q, r = divmod(npieces, mp)
        return q + (1 if r and not (q > 0 and mp + r <= (24 if bf16 else 32)) else 0)

    mp = _OVERRIDE_WIDTH()
    if not mp:
        mp = 24 if passes(24) < passes(16) and n_cols * 384 <= 96 << 20 else 16
    return (0 if reuse else 4) + passes(mp)


def _OVERRIDE_WIDTH():
    w = es._OVERRIDE["tune"][1]
    return w if w in (8, 16, 24) else 0


def _is_flow():
    return es._OVERRIDE["kernel"] in (es.ES_KERNEL_AUTO, es.ES_KERNEL_SLAB, es.ES_KERNEL_SLAB_FLOW)


def slab(rowptr, colind, val, B, s, strat, seed, reduce, F, **kw):
    ws = es.es_spmm_workspace(len(rowptr) - 1, B.shape[0], len(colind), F, B.shape[1], s, val is not None,
                              device=DEV)
    assert ws is not None
    vd = None if val is None else t(val)
    n0 = es.es_launch_count()
    if _unsupported_ok(B):
        with pytest.raises(es.EsError, match="UNSUPPORTED"):
            es.es_spmm_run_ex(t(rowptr), t(colind), vd, t(B), s, strat, seed, reduce, F=F, workspace=ws, **kw)
        with es.kernel_override("slab_smem"):
            return slab(rowptr, colind, val, B, s, strat, seed, reduce, F, **kw)
    out = es.es_spmm_run_ex(t(rowptr), t(colind), vd, t(B), s, strat, seed, reduce, F=F, workspace=ws,
                            **kw).cpu().numpy()
    assert es.es_spmm_workspace_status(ws) == es.ES_WS_OK
    # the slab path really ran (it launches the sampling kernels and/or one kernel per slice;
    # a silent fallback to the fused kernel would launch exactly one)
    if _is_flow():
        assert es.es_launch_count() - n0 == flow_launches(F), "flow path not taken"
    else:
        assert es.es_launch_count() - n0 >= (F + 63) // 64 + (0 if strat == 1 else 4) and \
            es.es_launch_count() - n0 > 1 or F <= 64, "slab path not taken"
    return out


@pytest.mark.parametrize("F,ld", [(17, 20), (64, 64), (65, 68), (200, 200), (602, 604), (602, 608)])
@pytest.mark.parametrize("strat", [1, 2])
def test_slab_parity(graph, lanes, F, ld, strat):
    rowptr, colind, val = graph
    B = synth.dense(2300, F, seed=F + 1, ld=ld)
    for s, seed, reduce in [(32, 0, 0), (256, 5, 1), (1000, 0, 1), (1, 3, 0), (100000, 2, 1)]:
        g = slab(rowptr, colind, val, B, s, strat, seed, reduce, F)
        o = oracle.spmm(rowptr, colind, val, B, s, strat, seed=seed, reduce=reduce, F=F)
        ok, err = rel_ok(g, o)
        assert ok, (F, ld, s, seed, reduce, err)


def test_slab_val_null_and_ones_exact(graph, lanes):
    """val NULL (no slot values stored) and B == 1: C = k_i exactly (SUM), 1 (MEAN)."""
    rowptr, colind, _ = graph
    d = np.diff(rowptr)
    B = np.ones((2300, 608), np.float32)
    for s in (1, 64, 700):
        for strat in (1, 2):
            g = slab(rowptr, colind, None, B, s, strat, 3, 0, 602)
            assert np.array_equal(g, np.repeat(np.minimum(d, s)[:, None], 602, 1).astype(np.float32))
            gm = slab(rowptr, colind, None, B, s, strat, 3, 1, 602)
            assert np.array_equal(gm, np.repeat((d > 0)[:, None], 602, 1).astype(np.float32))


def test_slab_options(graph, lanes):
    rowptr, colind, val = graph
    B = synth.dense(2300, 300, seed=9, ld=300)
    g = slab(rowptr, colind, val, B, 40, 2, 5, 1, 300, prime=7)
    o = oracle.spmm(rowptr, colind, val, B, 40, 2, seed=5, reduce=1, F=300, prime=7)
    assert rel_ok(g, o)[0]
    d = np.diff(rowptr)
    ones = np.ones((2300, 300), np.float32)
    g = slab(rowptr, colind, None, ones, 64, 2, 0, 1, 300, mean_by_degree=True)
    k = np.minimum(d, 64)
    want = np.where(d > 0, k.astype(np.float32) / np.maximum(d, 1).astype(np.float32), 0).astype(np.float32)
    assert np.array_equal(g, np.repeat(want[:, None], 300, 1))


def test_g16_is_bitwise_cpasync_hw(graph):
    """The documented order: with 16 lanes per slot the slab kernel sums exactly as the fused
    two-slots-per-step ring (spmm_cpasync_hw) does, so F <= 128 results are bitwise equal."""
    rowptr, colind, val = graph
    B = synth.dense(2300, 128, seed=4)
    with es.kernel_override("halfwarp"):
        fused = es.es_spmm_run(t(rowptr), t(colind), t(val), t(B), 256, 2, 7, 1, F=128).cpu().numpy()
    with es.kernel_override("slab_smem", 0, 16):
        g = slab(rowptr, colind, val, B, 256, 2, 7, 1, 128)
    assert np.array_equal(g, fused)


@pytest.mark.parametrize("F,ld", [(128, 128), (602, 608)])
def test_slab_kernels_same_order_bitwise(graph, F, ld):
    """The documented per-element order: the 8-lane shared-memory ring, the register-direct
    kernel (8 lanes x 32 B) on full slices and the TMA gather4 kernel all sum slot j into group
    j mod 4 in slot order, so full 64-float slices agree bitwise (the narrow last slice of F=602
    uses 4 lanes per slot in the first two, 8 in the TMA kernel)."""
    rowptr, colind, val = graph
    B = synth.dense(2300, F, seed=14, ld=ld)
    outs = {}
    for fam, tune in (("slab_smem", ()), ("slab_ldg", ()), ("slab_tma", ()), ("slab_stream", ()),
                      ("slab_flow", ()), ("slab_flow", (0, 16)), ("slab_flow", (8,))):
        with es.kernel_override(fam, *tune):
            outs[(fam,) + tune] = slab(rowptr, colind, val, B, 256, 2, 7, 1, F)
    full = (F // 64) * 64
    ref = outs[("slab_smem",)]
    assert np.array_equal(ref[:, :full], outs[("slab_ldg",)][:, :full])
    assert np.array_equal(ref[:, :full], outs[("slab_tma",)][:, :full])
    assert np.array_equal(ref, outs[("slab_stream",)])                    # same narrow-slice kernels too
    # the flow kernel: 8 lanes per slot for every slice width (no narrow-slice kernel), so it is
    # the TMA kernel's order on every column, whatever the slicing or CTA size
    for key in (("slab_flow",), ("slab_flow", 0, 16), ("slab_flow", 8)):
        assert np.array_equal(outs[key], outs[("slab_tma",)]), key


def test_slab_row_blocks_bitwise(graph, lanes):
    """Row blocks (es_spmm_run_ex on a CSR slice, global row ids) == the full launch, bitwise."""
    rowptr, colind, val = graph
    B = synth.dense(2300, 602, seed=8, ld=608)
    full = slab(rowptr, colind, val, B, 256, 2, 99, 1, 602)
    bounds = es.es_partition_rows(rowptr, 256, 602, 3)
    for a, b in zip(bounds[:-1], bounds[1:]):
        e0, e1 = int(rowptr[a]), int(rowptr[b])
        ws = es.es_spmm_workspace(int(b - a), 2300, e1 - e0, 602, 608, 256, True, device=DEV)
        part = es.es_spmm_run_ex(t(rowptr[a:b + 1]), t(colind[e0:e1]), t(val[e0:e1]), t(B), 256, 2, 99, 1,
                                 F=602, row_begin=int(a), row_end=int(b), n_rows=len(rowptr) - 1,
                                 nnz_base=e0, workspace=ws, nnz=e1 - e0).cpu().numpy()
        assert np.array_equal(part, full[a:b])


def test_slab_ldc_padding_untouched(graph, lanes):
    rowptr, colind, val = graph
    B = synth.dense(2300, 130, seed=2, ld=136)
    ws = es.es_spmm_workspace(1301, 2300, len(colind), 130, 136, 64, True, device=DEV)
    C = torch.full((1301, 140), -7.0, dtype=torch.float32, device=DEV)
    es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 64, 1, 0, 0, F=130, C=C, workspace=ws)
    Ch = C.cpu().numpy()
    assert np.all(Ch[:, 130:] == -7.0)
    o = oracle.spmm(rowptr, colind, val, B, 64, 1, F=130)
    assert rel_ok(Ch[:, :130], o)[0]


def test_auto_plan_choice():
    # Reddit-shaped F=602: B (566 MB) > L2, a 64-float slab (60 MB) fits -> workspace wanted
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 602, 608, 256) > 0
    # long rows with B L2-resident (Proteins-shaped) -> wanted; short rows (Arxiv-shaped), s < 32 for
    # F > 128, or a B too tall for any L2-resident slab (10M rows) -> none
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 602, 608, 64) > 0     # flow beats fused
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 602, 608, 16) == 0
    assert es.es_spmm_workspace_bytes(132534, 132534, 79_100_000, 128, 128, 256) > 0
    assert es.es_spmm_workspace_bytes(169343, 169343, 2_330_000, 128, 128, 64) == 0
    assert es.es_spmm_workspace_bytes(10_000_000, 10_000_000, 10**9, 256, 256, 128) == 0


def test_reuse_sampled_slots(graph, lanes):
    """reuse_sampled: the gather passes alone over the slots an earlier call sampled into the
    workspace (a second feature matrix over the same sampled graph) == a full call, bitwise."""
    rowptr, colind, val = graph
    B1 = synth.dense(2300, 300, seed=21, ld=304)
    B2 = synth.dense(2300, 300, seed=22, ld=304)
    ws = es.es_spmm_workspace(1301, 2300, len(colind), 300, 304, 96, True, device=DEV)
    rp, ci, v = t(rowptr), t(colind), t(val)
    es.es_spmm_run_ex(rp, ci, v, t(B1), 96, 2, 13, 1, F=300, workspace=ws)
    g2 = es.es_spmm_run_ex(rp, ci, v, t(B2), 96, 2, 13, 1, F=300, workspace=ws, reuse_sampled=True)
    full2 = slab(rowptr, colind, val, B2, 96, 2, 13, 1, 300)
    assert np.array_equal(g2.cpu().numpy(), full2)
    o = oracle.spmm(rowptr, colind, val, B2, 96, 2, seed=13, reduce=1, F=300)
    assert rel_ok(full2, o)[0]


def test_slab_launch_count(graph):
    """The launches es_launch_count reports (bench.py's gpu_launches) match the kernels the slab
    path runs: count + CUB scan (2 kernels) + materialise + one per 64-float slice; Bucket reads
    its slots in place (slices only); reuse_sampled runs the slices only."""
    with es.kernel_override("slab_smem"):
        _slab_launch_count(graph, ((2, False, 4 + 10), (1, False, 10), (2, True, 10)))
    # the flow kernel (the plan's): F = 602 is 151 16-B pieces -> 5 passes of 24 + one of 31
    # (the remainder merged); Bucket is materialised too (the padded layout)
    with es.kernel_override("slab"):
        _slab_launch_count(graph, ((2, False, 4 + 6), (1, False, 4 + 6), (2, True, 6)))
    with es.kernel_override("slab_flow", 0, 16):                # 8 x 16 + 23 merged
        _slab_launch_count(graph, ((2, False, 4 + 9), (2, True, 9)))


def _slab_launch_count(graph, cases):
    rowptr, colind, val = graph
    B = synth.dense(2300, 602, seed=1, ld=608)
    ws = es.es_spmm_workspace(1301, 2300, len(colind), 602, 608, 256, True, device=DEV)
    for strat, reuse, want in cases:
        n0 = es.es_launch_count()
        es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 256, strat, 0, 1, F=602, workspace=ws,
                          reuse_sampled=reuse)
        torch.cuda.synchronize()
        assert es.es_launch_count() - n0 == want, (strat, reuse)


# ------------------------------------------------------------------ workspace contract
def test_undersized_workspace_is_an_error(graph):
    """A workspace that cannot hold the sampled slots is ES_ERR_INVALID_VALUE (never a silent
    truncation), and so is one sized for val = NULL used with val."""
    rowptr, colind, val = graph
    B = synth.dense(2300, 602, seed=1, ld=608)
    full = es.es_spmm_workspace_bytes(1301, 2300, len(colind), 602, 608, 256, True, kernel="slab")
    small = torch.zeros(full // 2, dtype=torch.uint8, device=DEV)
    with es.kernel_override("slab"):
        with pytest.raises(es.EsError, match="INVALID"):
            es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 256, 2, 0, 1, F=602, workspace=small)
        noval = es.es_spmm_workspace(1301, 2300, len(colind), 602, 608, 256, False, device=DEV)
        with pytest.raises(es.EsError, match="INVALID"):
            es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 256, 2, 0, 1, F=602, workspace=noval)
        # sized for val = NULL, used with val = NULL: fine
        g = es.es_spmm_run_ex(t(rowptr), t(colind), None, t(B), 256, 2, 0, 1, F=602, workspace=noval)
        o = oracle.spmm(rowptr, colind, None, B, 256, 2, reduce=1, F=602)
        assert rel_ok(g.cpu().numpy(), o)[0]


def test_understated_nnz_poisons_rows_and_flags_overflow(graph):
    """The device backstop: a caller that understates nnz gets NaN rows for every row whose
    slots do not fit, and ES_WS_OVERFLOW in the workspace status -- never a truncated sum."""
    rowptr, colind, val = graph
    B = synth.dense(2300, 128, seed=2)
    k = np.minimum(np.diff(rowptr), 256)
    # the workspace bound includes the flow layout's padding slack (15 slots per row): state an
    # nnz that leaves the padded slots ~2,000 short
    kpad = int(((k + 15) // 16 * 16).sum())
    lie = max(1, kpad - 15 * 1301 - 2000)
    nb = es.es_spmm_workspace_bytes(1301, 2300, lie, 128, 128, 256, True, kernel="slab")
    ws = torch.zeros(nb, dtype=torch.uint8, device=DEV)
    with es.kernel_override("slab"):
        C = es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 256, 2, 0, 1, F=128, workspace=ws, nnz=lie)
    st = es.es_spmm_workspace_status(ws, reset=True)
    assert st & es.ES_WS_OVERFLOW
    g = C.cpu().numpy()
    bad = np.isnan(g).all(axis=1)
    assert bad.any() and not bad.all()
    assert not np.isnan(g[~bad]).any()
    # rows are materialised in order: exactly the rows whose slots end past the capacity -- a
    # suffix of the rows -- are poisoned
    r0 = int(np.argmax(bad))
    assert bad[r0:].all() and not bad[:r0].any()
    fine = ~bad
    o = oracle.spmm(rowptr, colind, val, B, 256, 2, reduce=1, F=128)
    assert rel_ok(g[fine], o[fine])[0]
    assert es.es_spmm_workspace_status(ws) == es.ES_WS_OK          # reset


def test_reuse_with_other_sampling_is_detected(graph):
    """reuse_sampled over slots of a different sampling (other seed / s / graph): NaN rows and
    ES_WS_SIGNATURE_MISMATCH; a layout that cannot take the slab path refuses reuse."""
    rowptr, colind, val = graph
    B = synth.dense(2300, 300, seed=3, ld=300)
    ws = es.es_spmm_workspace(1301, 2300, len(colind), 300, 300, 96, True, device=DEV, kernel="slab")
    rp, ci, v = t(rowptr), t(colind), t(val)
    with es.kernel_override("slab"):
        es.es_spmm_run_ex(rp, ci, v, t(B), 96, 2, 13, 1, F=300, workspace=ws)
        assert es.es_spmm_workspace_status(ws) == es.ES_WS_OK
        # a re-uploaded copy of the same graph may reuse the slots; a different graph (same row
        # count, other degrees) is caught row by row
        C = es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 96, 2, 13, 1, F=300, workspace=ws,
                              reuse_sampled=True)
        assert not torch.isnan(C).any() and es.es_spmm_workspace_status(ws) == es.ES_WS_OK
        rp2 = rowptr.copy()
        rp2[1:-1] = np.minimum(rp2[1:-1] + 1, rp2[-1])     # shifted row boundaries
        C = es.es_spmm_run_ex(t(rp2), ci, v, t(B), 96, 2, 13, 1, F=300, workspace=ws, reuse_sampled=True)
        assert torch.isnan(C).any()
        assert es.es_spmm_workspace_status(ws, reset=True) & es.ES_WS_SIGNATURE_MISMATCH
        for kw in (dict(seed=14), dict(s=95)):
            args = dict(seed=13, s=96)
            args.update(kw)
            C = es.es_spmm_run_ex(rp, ci, v, t(B), args["s"], 2, args["seed"], 1, F=300, workspace=ws,
                                  reuse_sampled=True)
            assert torch.isnan(C).all()
            assert es.es_spmm_workspace_status(ws, reset=True) & es.ES_WS_SIGNATURE_MISMATCH
        C = es.es_spmm_run_ex(rp, ci, v, t(B), 96, 2, 13, 1, F=300, workspace=ws, reuse_sampled=True)
        assert not torch.isnan(C).any()
    # unaligned B rows: no slab path, so nothing to reuse -> error, not a silent fused run
    B2 = t(synth.dense(2300, 301, seed=3, ld=301))
    with pytest.raises(es.EsError, match="INVALID"):
        es.es_spmm_run_ex(rp, ci, v, B2, 96, 2, 13, 1, F=301, workspace=ws, reuse_sampled=True)


# ------------------------------------------------------------------ flow kernel specifics
@pytest.mark.parametrize("case", ["short", "empty_batches", "one_long_row", "all_empty", "few_rows"])
def test_flow_row_structure(case):
    """The flow kernel's stream bookkeeping: rows of every length mod 4 (padding), runs of more
    than 32 empty rows (whole metadata batches with nothing to stream), one row holding most of
    the slots (the slot-balanced partition puts it alone), a graph with no edges, and fewer rows
    than warps -- every row against the oracle, bitwise equal to the per-row TMA gather4 kernel
    (the same per-element order)."""
    rng = np.random.default_rng(7)
    n_cols = 3000
    if case == "short":
        d = rng.integers(0, 23, 5000)
    elif case == "empty_batches":
        d = rng.integers(1, 40, 4000)
        d[100:190] = 0
        d[1000:1033] = 0
        d[3900:] = 0
    elif case == "one_long_row":
        d = rng.integers(0, 5, 3000)
        d[1500] = 2999
    elif case == "all_empty":
        d = np.zeros(777, np.int64)
    else:
        d = rng.integers(0, 300, 37)
    rowptr = np.zeros(len(d) + 1, np.int64)
    np.cumsum(d, out=rowptr[1:])
    colind = synth.columns(rowptr, n_cols, np.ones(n_cols, np.int64), 11) if rowptr[-1] else np.zeros(0, np.int32)
    val = (rng.random(len(colind), dtype=np.float32) + 0.5).astype(np.float32)
    B = synth.dense(n_cols, 602, seed=3, ld=608)
    for s, strat, reduce in ((256, 2, 1), (7, 1, 0), (3000, 2, 0)):
        with es.kernel_override("slab_flow"):
            g = slab(rowptr, colind, val, B, s, strat, 5, reduce, 602)
        o = oracle.spmm(rowptr, colind, val, B, s, strat, seed=5, reduce=reduce, F=602)
        ok, err = rel_ok(g, o)
        assert ok, (case, s, err)
        with es.kernel_override("slab_tma"):
            ref = slab(rowptr, colind, val, B, s, strat, 5, reduce, 602)
        assert np.array_equal(g, ref), case


def test_flow_bf16_parity(graph):
    """bf16 storage of B (NEXT-4) on the flow kernel: slices of <= 16 pieces (128 elements)."""
    rowptr, colind, val = graph
    Bf = synth.dense(2300, 602, seed=5, ld=608)
    Bb = torch.from_numpy(Bf).to(DEV).to(torch.bfloat16)
    Bw = Bb.float().cpu().numpy()                       # the exactly widened values
    ws = es.es_spmm_workspace(1301, 2300, len(colind), 602, 608, 256, True, device=DEV, kernel="slab")
    n0 = es.es_launch_count()
    g = es.es_spmm_run_ex(t(rowptr), t(colind), t(val), Bb, 256, 2, 3, 1, F=602, workspace=ws, kernel="slab")
    torch.cuda.synchronize()
    assert es.es_launch_count() - n0 == flow_launches(602, bf16=True)
    o = oracle.spmm(rowptr, colind, val, Bw, 256, 2, seed=3, reduce=1, F=602)
    assert rel_ok(g.cpu().numpy(), o)[0]
