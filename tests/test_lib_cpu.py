"""The C-ABI library loads and exports every symbol include/es_spmm.h declares; host-side
logic (validation, partitioner, plan) works without a GPU.  No compute calls here."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2104_10716_b200 as es
from paper_2104_10716_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return es.load_library()


def test_header_declarations_are_exported(lib):
    with open(os.path.join(ROOT, "include", "es_spmm.h")) as f:
        text = f.read()
    declared = set(re.findall(r"^\s*(?:es_status_t|int64_t|int32_t|void|const char\*)\s+(es_\w+)\s*\(", text, re.M))
    assert declared == set(es.EXPORTS), declared ^ set(es.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    # the sm_100a cubin is embedded
    blob = open(es.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob or b"sm_100" in blob


def test_status_strings(lib):
    assert es.es_status_string(0) == "ES_OK"
    assert es.es_status_string(1) == "ES_ERR_INVALID_VALUE"
    assert es.es_status_string(4) == "ES_ERR_CUDA"


def test_host_validation_rejects_bad_arguments(lib):
    vp = ctypes.c_void_p
    dummy = vp(16)
    ok = dict(n_rows=10, n_cols=10, F=8, ldb=8, s=4, strategy=2, reduce=0, ldc=8)

    def run(**kw):
        a = dict(ok, **kw)
        return lib.es_spmm_run(a["n_rows"], a["n_cols"], dummy, dummy, None, dummy, a["F"], a["ldb"],
                               a["s"], a["strategy"], 0, a["reduce"], dummy, a["ldc"], None)

    assert run(s=0) == es.ES_ERR_INVALID_VALUE
    assert run(F=0) == es.ES_ERR_INVALID_VALUE
    assert run(ldb=7) == es.ES_ERR_INVALID_VALUE
    assert run(ldc=7) == es.ES_ERR_INVALID_VALUE
    assert run(strategy=3) == es.ES_ERR_INVALID_VALUE
    assert run(reduce=2) == es.ES_ERR_INVALID_VALUE
    assert run(n_rows=-1) == es.ES_ERR_INVALID_VALUE
    assert run(n_rows=0) == es.ES_OK          # nothing to launch
    # NULL required pointers
    assert lib.es_spmm_run(10, 10, None, dummy, None, dummy, 8, 8, 4, 2, 0, 0, dummy, 8, None) == 1
    assert lib.es_spmm_run(10, 10, dummy, dummy, None, dummy, 8, 8, 4, 2, 0, 0, None, 8, None) == 1
    # row range checks
    assert lib.es_spmm_run_rows(10, 10, dummy, 0, dummy, None, dummy, 8, 8, 4, 2, 0, 0, dummy, 8,
                                5, 11, None) == 1
    assert lib.es_spmm_run_rows(10, 10, dummy, 0, dummy, None, dummy, 8, 8, 4, 2, 0, 0, dummy, 8,
                                6, 5, None) == 1
    assert lib.es_spmm_sample(10, 10, dummy, dummy, None, 0, 2, 0, 0, dummy, None, None, None,
                              None) == 1
    assert lib.es_spmm_sample(10, 10, dummy, dummy, None, 3, 9, 0, 0, dummy, None, None, None,
                              None) == 1


def test_plan_selection(lib):
    assert es.es_spmm_plan(128, 128, 128).startswith("es::spmm_segstream<rows8>")
    assert es.es_spmm_plan(200, 200, 200).startswith("es::spmm_cpasync<stages4>")
    assert es.es_spmm_plan(256, 256, 256).startswith("es::spmm_cpasync<stages4>")
    assert es.es_spmm_plan(512, 512, 512).startswith("es::spmm_cpasync<stages4>")
    assert es.es_spmm_plan(602, 604, 604).startswith("es::spmm_tma<nch5,stages4>")
    assert es.es_spmm_plan(100, 102, 100).startswith("es::spmm_warp<vec2")      # 8-B aligned rows
    assert "spmm_warp<vec2" in es.es_spmm_plan(602, 602, 602)      # 8-B rows: no TMA
    assert "subwarp<vec4,g4>" in es.es_spmm_plan(16, 16, 16)
    assert "subwarp<vec1,g1>" in es.es_spmm_plan(1, 1, 1)
    assert "spmm_warp<vec4,nch8>" in es.es_spmm_plan(5000, 5000, 5000)   # feature-tiled


def test_product_library_reads_no_environment():
    """Kernel selection arrives through es_spmm_options_t only: the
    library's sources call no getenv (the statically linked CUDA runtime reads its own
    CUDA_* variables; that is not ours)."""
    csrc = os.path.join(ROOT, "paper_2104_10716_b200", "csrc")
    for f in os.listdir(csrc):
        if f.endswith((".cu", ".cuh", ".h")):
            assert "getenv" not in open(os.path.join(csrc, f)).read(), f


def test_forced_kernel_option_is_validated(lib):
    Opt = es.EsOptions
    dummy = ctypes.c_void_p(0x1000)
    bad = Opt.make()
    bad.kernel = 42
    assert lib.es_spmm_run_ex(10, 10, dummy, 0, dummy, None, dummy, 8, 8, 4, 2, 0, 0, dummy, 8, 0, 10,
                              ctypes.byref(bad), None) == es.ES_ERR_INVALID_VALUE
    # a slab kernel forced without a workspace: the path cannot run
    assert lib.es_spmm_run_ex(10, 10, dummy, 0, dummy, None, dummy, 8, 8, 4, 2, 0, 0, dummy, 8, 0, 10,
                              ctypes.byref(Opt.make(kernel="slab")), None) == es.ES_ERR_UNSUPPORTED


def test_undersized_workspace_rejected_on_host(lib):
    """The capacity check is host arithmetic (no device access): a workspace that cannot hold
    min(nnz, n*s) slots -- or n*s when nnz is not stated -- is ES_ERR_INVALID_VALUE."""
    Opt = es.EsOptions
    dummy = ctypes.c_void_p(0x1000)
    n, s, F, ldb = 1000, 64, 602, 608
    need = es.es_spmm_workspace_bytes(n, n, 20000, F, ldb, s, True, kernel="slab")

    class _T:                                       # a stand-in "tensor" for EsOptions.make
        def __init__(self, nbytes):
            self.n = nbytes

        def numel(self):
            return self.n

        def element_size(self):
            return 1

        def data_ptr(self):
            return 0x100000

    def run(nbytes, nnz, val=dummy):
        o = Opt.make(workspace=_T(nbytes), nnz=nnz, kernel="slab")
        return lib.es_spmm_run_ex(n, n, dummy, 0, dummy, val, ctypes.c_void_p(0x2000), F, ldb, s, 2, 0, 1,
                                  ctypes.c_void_p(0x3000), ldb, 0, n, ctypes.byref(o), None)
    assert run(need - 4096, 20000) == es.ES_ERR_INVALID_VALUE          # too small for nnz slots
    assert run(need, 0) == es.ES_ERR_INVALID_VALUE                     # nnz unknown: n*s = 64000 slots
    noval = es.es_spmm_workspace_bytes(n, n, 20000, F, ldb, s, False, kernel="slab")
    assert run(noval, 20000) == es.ES_ERR_INVALID_VALUE                # sized for val NULL, val passed


class _B:
    def __init__(self, p):
        self.p = p

    def data_ptr(self):
        return self.p


def test_plan_alignment_fallback(lib):
    # B misaligned by 4 bytes -> scalar gathers; C misaligned -> scalar stores
    assert "vec1" in es.es_spmm_plan(128, 128, 128, B=_B(0x1004), C=_B(0x1000))
    assert "vec2" in es.es_spmm_plan(128, 128, 128, B=_B(0x1008), C=_B(0x1000))
    assert "scalar C" in es.es_spmm_plan(128, 128, 128, B=_B(0x1000), C=_B(0x1004))


def _ref_bounds(rowptr, s, F, P):
    d = np.diff(rowptr)
    w = np.minimum(d, s) * (4 * F + 8) + 4 * F
    pre = np.concatenate([[0], np.cumsum(w)])
    tot = int(pre[-1])
    out = [0]
    for p in range(1, P):
        tgt = -(-tot * p // P)
        r = int(np.searchsorted(pre, tgt, side="left"))
        out.append(max(min(r, len(d)), out[-1]))
    out.append(len(d))
    return np.array(out)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_rows(lib, P):
    rng = np.random.default_rng(P)
    d = np.minimum((rng.pareto(1.1, 5000) * 20).astype(np.int64), 20000)
    rowptr = np.concatenate([[0], np.cumsum(d)])
    for s, F in [(256, 602), (16, 128), (10**9, 64)]:
        b = es.es_partition_rows(rowptr, s, F, P)
        assert b[0] == 0 and b[-1] == 5000 and np.all(np.diff(b) >= 0)
        assert np.array_equal(b, _ref_bounds(rowptr, s, F, P))
        # balance: every part within one max-row weight of the ideal share
        w = np.minimum(d, s) * (4 * F + 8) + 4 * F
        parts = [w[b[i]:b[i + 1]].sum() for i in range(P)]
        assert max(parts) - w.sum() / P <= w.max()
    # with s >= max degree the weights are nnz-proportional (+ per-row constant)
    b = es.es_partition_rows(rowptr, 10**9, 1, P)
    assert np.array_equal(b, _ref_bounds(rowptr, 10**9, 1, P))


def test_partition_degenerate(lib):
    assert es.es_partition_rows(np.zeros(1, np.int64), 4, 8, 3).tolist() == [0, 0, 0, 0]
    assert es.es_partition_rows(np.array([0, 5], np.int64), 4, 8, 4).tolist()[-1] == 1


def test_options_validation(lib):
    vp = ctypes.c_void_p
    dummy = vp(16)
    Opt = es.EsOptions

    def run(opt, ldb=8, F=8, B=dummy):
        return lib.es_spmm_run_ex(10, 10, dummy, 0, dummy, None, B, F, ldb, 4, 2, 0, 0, dummy, F, 0, 10,
                                  ctypes.byref(opt), None)

    assert run(Opt(4, 0, 0, 0)) == es.ES_ERR_INVALID_VALUE                 # struct_size too small
    assert run(Opt(ctypes.sizeof(Opt), -3, 0, 0)) == es.ES_ERR_INVALID_VALUE
    assert run(Opt(ctypes.sizeof(Opt), 0, 2, 0)) == es.ES_ERR_INVALID_VALUE
    assert run(Opt(ctypes.sizeof(Opt), 0, 0, 7)) == es.ES_ERR_INVALID_VALUE
    # bf16 needs 16-B rows: ldb % 8 != 0 or a misaligned B -> unsupported (decided before launch)
    assert run(Opt.make(bf16=True), ldb=12, F=12) == es.ES_ERR_UNSUPPORTED
    assert run(Opt.make(bf16=True), ldb=16, F=16, B=vp(0x1008)) == es.ES_ERR_UNSUPPORTED
    # backward has no bf16 variant
    assert lib.es_spmm_backward_ex(10, 10, dummy, 0, dummy, None, dummy, 8, 8, 4, 2, 0, 0, dummy, 8, 0, 10,
                                   ctypes.byref(Opt.make(bf16=True)), None) == es.ES_ERR_UNSUPPORTED


def test_workspace_bytes_plan(lib):
    """es_spmm_workspace_bytes (host only): the slab path is asked for when a 64-float slab of B
    fits L2, F >= 128, ldb % 4 == 0 and rows sample enough slots on average; the bound covers
    min(nnz, n*s) slots plus the flow layout's padding (<= 15 slots per row) (+ values) and each
    row's unpadded k_i."""
    reddit = es.es_spmm_workspace_bytes(232965, 232965, 114615945, 602, 608, 256)
    assert reddit >= 8 * 232965 * 256 + 8 * 232966            # n*s < nnz here: n*s slots
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 602, 608, 256, has_val=False) < reddit
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 128, 128, 256) > 0     # B 119 MB
    assert es.es_spmm_workspace_bytes(132534, 132534, 79_100_000, 128, 128, 256) > 0    # long rows
    assert es.es_spmm_workspace_bytes(169343, 169343, 2_330_000, 128, 128, 64) == 0     # short rows
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 128, 128, 128) == 0    # F <= 128: fused below s = 256
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 256, 256, 128) > 0     # 128 < F <= 256: from s = 128
    assert es.es_spmm_workspace_bytes(10_000_000, 10_000_000, 10**9, 256, 256, 128) == 0  # slab > L2
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 64, 64, 256) == 0      # one slice
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 602, 608, 64) > 0      # s >= 32, F > 128
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 602, 608, 16) == 0     # s < 32
    assert es.es_spmm_workspace_bytes(232965, 232965, 114615945, 602, 602, 256) == 0    # 8-B row pitch
    small = es.es_spmm_workspace_bytes(232965, 232965, 1000, 602, 608, 256, kernel="slab")
    n = 232965
    assert 8 * (1000 + 15 * n) + 4 * n <= small - 8 * (n + 1) < 8 * (1000 + 15 * n) + 4 * n + 8192  # nnz < n*s
    assert es.es_spmm_workspace_bytes(10, 10, 10, 602, 600, 4) == 0                     # ldb < F
    assert es.es_spmm_workspace_bytes(100, 100, 1000, 602, 608, 256, kernel="slab") > 0
