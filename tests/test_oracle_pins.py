"""Pins for the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names what it pins and why a plausible oracle bug (dropped term, wrong
sign/index, transposed operand, wrong divisor, wrong row id in the seeded offset)
would fail it.  Oracle functions pinned here: mix64/offset, position, rate, sample,
spmm (SUM/MEAN, Bucket/FastRand, seeded, row subsets, row_base), spmm_backward (adjoint
identity, dense brute force, column-hit counts) and brute.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth
from oracle import BUCKET, FASTRAND, SUM, MEAN


# ----------------------------------------------------------------- Eq. 2 positions
def test_fastrand_index_spec_examples(golden):
    for j, d, want in golden["fastrand_index"]["cases"]:
        assert oracle.position(FASTRAND, j, d) == want


def test_sample_row_spec_example(golden):
    g = golden["sample_row"]
    d = len(g["cols"])
    pos = [oracle.position(FASTRAND, j, d) for j in range(min(d, g["s"]))]
    assert pos == g["positions"]
    assert [g["cols"][p] for p in pos] == g["sampled_cols"]
    assert [oracle.position(FASTRAND, j, 10) for j in range(10)] == \
        golden["full_row_permutation_d10"]["positions"]


def test_fastrand_is_permutation_iff_577_does_not_divide_d():
    # 577 is prime: j -> 577 j mod d is a bijection of Z_d iff gcd(577, d) = 1.
    for d in list(range(1, 1300)) + [577 * 3, 577 * 4 + 1, 4999]:
        ps = [oracle.position(FASTRAND, j, d) for j in range(d)]
        assert all(0 <= p < d for p in ps)
        if d % 577:
            assert sorted(ps) == list(range(d)), d
        else:
            m = d // 577  # positions cycle with period m through multiples of 577
            assert ps[:m] == [(577 * j) % d for j in range(m)]
            assert ps[m:2 * m] == ps[:m]
            assert len(set(ps)) == m


def test_fastrand_special_residues():
    # d | 576  =>  577 = 1 (mod d): FastRand order == Bucket order.
    for d in [1, 2, 3, 4, 6, 8, 9, 12, 16, 18, 24, 32, 36, 48, 64, 72, 96, 144, 192, 288, 576]:
        assert [oracle.position(FASTRAND, j, d) for j in range(d)] == list(range(d))
    # d | 578  =>  577 = -1 (mod d): positions 0, d-1, d-2, ...
    for d in [17, 34, 289, 578]:
        assert [oracle.position(FASTRAND, j, d) for j in range(d)] == [(-j) % d for j in range(d)]
    # d > 577 (k-1): strictly increasing stride-577 progression.
    d, k = 577 * 9 + 5, 10
    assert [oracle.position(FASTRAND, j, d) for j in range(k)] == [577 * j for j in range(k)]


def test_position_large_values_no_overflow():
    # 64-bit intermediate: j * 577 >= 2^32 for j >= 7,443,617.
    for j, d in [(7_443_617, 2**31 - 1), (10**9, 10**12 + 39), (2**40, 2**41 + 1)]:
        assert oracle.position(FASTRAND, j, d) == (j * 577) % d


def test_random_pairs_against_python_bigint():
    rng = np.random.default_rng(9)
    js = rng.integers(0, 2**31, 2000)
    ds = rng.integers(1, 2**31, 2000)
    for j, d in zip(js.tolist(), ds.tolist()):
        assert oracle.position(FASTRAND, j, d) == (j * 577) % d


def test_bucket_positions():
    assert [oracle.position(BUCKET, j, 50) for j in range(7)] == list(range(7))


# ----------------------------------------------------------------- seeded offset (reading R6)
def test_seeded_offset_vectors(golden):
    g = golden["seeded_offset"]
    assert oracle.mix64(1) == int(g["mix64_1"], 16)
    assert [oracle.offset(g["seed"], r, g["d"]) for r in range(4)] == g["offsets"]
    off = oracle.offset(g["seed"], 0, g["d"])
    assert [oracle.position(FASTRAND, j, g["d"], off) for j in range(3)] == g["row0_s3_positions"]
    assert oracle.offset(0, 5, 10) == 0          # seed 0 is exactly Eq. 2
    assert oracle.offset(123, 5, 0) == 0


def test_seeded_offset_is_a_rotation():
    # A rotation keeps counts, distinctness and the selected multiset size.
    for d in [10, 97, 577, 1000, 1154]:
        for row in range(5):
            off = oracle.offset(77, row, d)
            assert 0 <= off < d
            base = [oracle.position(FASTRAND, j, d) for j in range(d)]
            rot = [oracle.position(FASTRAND, j, d, off) for j in range(d)]
            assert rot == [(off + b) % d for b in base]
            assert len(set(rot)) == len(set(base))


# ----------------------------------------------------------------- sampling rate (Table sample_rate)
def test_rate_spec_example(golden):
    g = golden["sampling_rate"]
    rowptr = np.concatenate([[0], np.cumsum(g["degrees"])])
    assert oracle.rate(rowptr, g["s"]) == pytest.approx(g["rate"], abs=0)
    assert oracle.rate(np.zeros(4, np.int64), 3) == 1.0      # nnz = 0 -> 1.0
    assert oracle.rate(rowptr, 9) == 1.0                     # s >= max degree


@pytest.mark.parametrize("name", ["pubmed", "arxiv", "proteins", "reddit"])
def test_rate_reproduces_table_sample_rate(golden, name):
    """The synthetic degree sequences reproduce every printed cell of Table sample_rate
     to its last digit; pins oracle.rate and the generator."""
    t = golden["sample_rate_table"]
    d = synth.degrees(name)
    rowptr = np.concatenate([[0], np.cumsum(d)])
    for s, pct in zip(t["s"], t[name]):
        r = oracle.rate(rowptr, s)
        assert abs(100 * r - pct) <= 0.05 + 1e-9, (name, s, 100 * r, pct)
    # monotone in s
    rs = [oracle.rate(rowptr, s) for s in [1, 2, 4, 16, 64, 256, 1024, 10**6]]
    assert all(a <= b for a, b in zip(rs, rs[1:])) and rs[-1] == 1.0
    assert oracle.rate(rowptr, 1) == pytest.approx(np.count_nonzero(d) / d.sum())


# ----------------------------------------------------------------- sample (materialised)
def test_sample_counts_positions_and_strategy_invariance():
    rowptr, colind, val = synth.random_csr(300, 2000, seed=3, max_deg=700,
                                           special=(577, 1154, 578, 576, 1))
    d = np.diff(rowptr)
    for s in [1, 2, 7, 32, 600, 5000]:
        K = int(np.minimum(d, s).sum())
        for strat in (BUCKET, FASTRAND):
            for seed in (0, 11):
                srp, sc, sv, spos = oracle.sample(rowptr, colind, val, s, strat, seed)
                assert np.array_equal(np.diff(srp), np.minimum(d, s))      # k_i = min(d_i, s)
                assert srp[-1] == K                                         # same for both strategies
                assert oracle.rate(rowptr, s) == pytest.approx(K / d.sum(), abs=0)
                for i in range(0, 300, 7):
                    ps = spos[srp[i]:srp[i + 1]].tolist()
                    assert ps == oracle.brute.positions(strat, int(d[i]), s, seed, i)
                    e = rowptr[i] + spos[srp[i]:srp[i + 1]]
                    assert np.array_equal(sc[srp[i]:srp[i + 1]], colind[e])
                    assert np.array_equal(sv[srp[i]:srp[i + 1]], val[e])


def test_sample_duplicates_kept_in_slot_order():
    d = 1154                                              # 577 | d: positions 0, 577, 0, 577, ...
    rowptr = np.array([0, d], np.int64)
    colind = np.arange(d, dtype=np.int32)
    srp, sc, sv, spos = oracle.sample(rowptr, colind, None, 6, FASTRAND)
    assert spos.tolist() == [0, 577, 0, 577, 0, 577]
    assert sv.tolist() == [1.0] * 6                       # val NULL -> 1.0


# ----------------------------------------------------------------- SpMM values
def _hand_case(g, c):
    strat = BUCKET if c["strategy"] == "bucket" else FASTRAND
    red = SUM if c["reduce"] == "sum" else MEAN
    B = np.array([[j + 1, 10 * (j + 1)] for j in range(g["n_cols"])], np.float32)
    return oracle.spmm(g["rowptr"], g["colind"], None, B, c["s"], strat, reduce=red), strat


def test_hand_golden(golden):
    g = golden["hand"]
    for c in g["cases"]:
        C, strat = _hand_case(g, c)
        assert np.array_equal(C, np.array(c["C"], np.float32)), c
        if "cols" in c:
            srp, sc, _, _ = oracle.sample(g["rowptr"], g["colind"], None, c["s"], strat)
            got = [sc[srp[i]:srp[i + 1]].tolist() for i in range(len(g["rowptr"]) - 1)]
            assert got == c["cols"]


def test_spec_spmm_examples(golden):
    g = golden["spmm_spec"]
    B = np.array(g["B"], np.float32)
    for strat in (BUCKET, FASTRAND):
        assert np.array_equal(oracle.spmm(g["rowptr"], g["colind"], g["val"], B, 100, strat),
                              np.array(g["exact"], np.float32))
        assert np.array_equal(oracle.spmm(g["rowptr"], g["colind"], g["val"], B, 1, strat),
                              np.array(g["bucket_s1"], np.float32))
    m = golden["gnn_mean_spec"]
    assert np.array_equal(oracle.spmm(m["rowptr"], m["colind"], None, np.array(m["B"], np.float32),
                                      8, BUCKET, reduce=MEAN), np.array(m["mean"], np.float32))


def _ulp_close(a, b, ulps=1):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    tol = ulps * np.spacing(np.maximum(np.abs(a), np.abs(b)).astype(np.float32))
    return np.all(np.abs(a.astype(np.float64) - b.astype(np.float64)) <= tol)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_s_ge_maxdeg_equals_scipy_exact(seed):
    """s >= max degree reproduces exact SpMM: Bucket against
    scipy.sparse (a library routine, fp64, stored order), FastRand likewise on rows
    coprime to 577 (same multiset of terms)."""
    rowptr, colind, val = synth.random_csr(400, 900, seed=seed, max_deg=300)
    B = synth.dense(900, 37, seed=seed + 100)
    A = sp.csr_matrix((val.astype(np.float64), colind, rowptr), shape=(400, 900))
    exact = (A @ B.astype(np.float64)).astype(np.float32)
    s = int(np.diff(rowptr).max()) + 1
    Cb = oracle.spmm(rowptr, colind, val, B, s, BUCKET)
    Cf = oracle.spmm(rowptr, colind, val, B, s, FASTRAND)
    Cfs = oracle.spmm(rowptr, colind, val, B, s, FASTRAND, seed=99)
    assert _ulp_close(Cb, exact)
    assert _ulp_close(Cf, exact)
    assert _ulp_close(Cfs, exact)
    # mean = exact / degree on non-empty rows
    d = np.diff(rowptr)
    Cm = oracle.spmm(rowptr, colind, val, B, s, BUCKET, reduce=MEAN)
    nz = d > 0
    assert _ulp_close(Cm[nz], (exact[nz] / d[nz, None].astype(np.float32)), ulps=2)
    assert np.all(Cm[~nz] == 0)


@pytest.mark.parametrize("strat", [BUCKET, FASTRAND])
@pytest.mark.parametrize("seed", [0, 5])
@pytest.mark.parametrize("reduce", [SUM, MEAN])
def test_against_dense_brute_force(strat, seed, reduce):
    rowptr, colind, val = synth.random_csr(60, 1300, seed=7 + seed, max_deg=40,
                                           special=(577, 1154, 578, 1200))
    B = synth.dense(1300, 9, seed=3)
    for s in [1, 3, 16, 600]:
        want = oracle.brute.spmm(rowptr, colind, val, B, s, strat, seed, reduce)
        got = oracle.spmm(rowptr, colind, val, B, s, strat, seed=seed, reduce=reduce)
        assert _ulp_close(got, want), (s, np.abs(got - want).max())


def test_ones_give_counts_exactly():
    """B == 1, val == 1, SUM: C[i, :] = k_i exactly (duplicates counted); MEAN: 1 or 0."""
    rowptr, colind, _ = synth.random_csr(200, 3000, seed=21, max_deg=900, special=(577, 1154, 1731))
    d = np.diff(rowptr)
    B = np.ones((3000, 5), np.float32)
    for s in [1, 4, 100, 1000]:
        for strat in (BUCKET, FASTRAND):
            C = oracle.spmm(rowptr, colind, None, B, s, strat, seed=3)
            assert np.array_equal(C, np.repeat(np.minimum(d, s)[:, None], 5, 1).astype(np.float32))
            Cm = oracle.spmm(rowptr, colind, None, B, s, strat, seed=3, reduce=MEAN)
            assert np.array_equal(Cm, np.repeat((d > 0)[:, None], 5, 1).astype(np.float32))


def test_s1_is_single_product():
    rowptr, colind, val = synth.random_csr(100, 500, seed=4)
    B = synth.dense(500, 12, seed=8)
    d = np.diff(rowptr)
    for strat in (BUCKET, FASTRAND):
        C = oracle.spmm(rowptr, colind, val, B, 1, strat)
        for i in range(100):
            if d[i]:
                e = rowptr[i]
                assert np.array_equal(C[i], val[e] * B[colind[e]])
            else:
                assert np.all(C[i] == 0)


def test_mean_divides_by_sampled_count_not_degree():
    # one row of degree 10, s = 4: mean over the 4 kept B rows (reading R5)
    rowptr = np.array([0, 10], np.int64)
    colind = np.arange(10, dtype=np.int32)
    B = np.arange(10, dtype=np.float32)[:, None] * np.float32(4.0)
    C = oracle.spmm(rowptr, colind, None, B, 4, BUCKET, reduce=MEAN)
    assert C[0, 0] == np.float32((0 + 4 + 8 + 12) / 4)


def test_feature_column_permutation_and_row_subsets():
    rowptr, colind, val = synth.random_csr(150, 700, seed=12, max_deg=90)
    B = synth.dense(700, 20, seed=5)
    perm = np.random.default_rng(0).permutation(20)
    for strat in (BUCKET, FASTRAND):
        C = oracle.spmm(rowptr, colind, val, B, 16, strat, seed=4, reduce=MEAN)
        Cp = oracle.spmm(rowptr, colind, val, np.ascontiguousarray(B[:, perm]), 16, strat, seed=4,
                         reduce=MEAN)
        assert np.array_equal(Cp, C[:, perm])
        rows = np.array([149, 0, 3, 77, 77], np.int64)
        assert np.array_equal(oracle.spmm(rowptr, colind, val, B, 16, strat, seed=4, reduce=MEAN,
                                          rows=rows), C[rows])
        # F < ldb uses only the first F columns
        assert np.array_equal(oracle.spmm(rowptr, colind, val, B, 16, strat, seed=4, reduce=MEAN,
                                          F=7), C[:, :7])


def test_row_slice_with_row_base_matches_global():
    """A row block [a, b) evaluated with row_base = a (the multi-GPU slice) equals
    rows a..b of the global evaluation bitwise (seeded offset uses the global row id)."""
    rowptr, colind, val = synth.random_csr(500, 800, seed=2, max_deg=120)
    B = synth.dense(800, 8, seed=1)
    full = oracle.spmm(rowptr, colind, val, B, 20, FASTRAND, seed=42)
    a, b = 123, 377
    part = oracle.spmm(rowptr[a:b + 1], colind, val, B, 20, FASTRAND, seed=42, row_base=a)
    assert np.array_equal(part, full[a:b])
    wrong = oracle.spmm(rowptr[a:b + 1], colind, val, B, 20, FASTRAND, seed=42, row_base=0)
    assert not np.array_equal(wrong, full[a:b])


def test_empty_inputs():
    B = synth.dense(5, 3, seed=1)
    C = oracle.spmm(np.zeros(1, np.int64), np.zeros(0, np.int32), None, B, 4, FASTRAND)
    assert C.shape == (0, 3)
    C = oracle.spmm(np.zeros(4, np.int64), np.zeros(0, np.int32), None, B, 4, FASTRAND, reduce=MEAN)
    assert C.shape == (3, 3) and np.all(C == 0)


# ----------------------------------------------------------------- backward (NEXT-2)
@pytest.mark.parametrize("strat", [BUCKET, FASTRAND])
@pytest.mark.parametrize("reduce", [SUM, MEAN])
def test_backward_adjoint_identity(strat, reduce):
    """<A_s B, dC> = <B, A_s^T dC>: the backward is the adjoint of the forward over the same
    sampled slots (a wrong index, a transposed operand or a missing 1/k breaks it)."""
    rowptr, colind, val = synth.random_csr(250, 400, seed=8, max_deg=120, special=(577, 1154 // 3))
    B = synth.dense(400, 11, seed=2)
    dC = synth.dense(250, 11, seed=3)
    C = oracle.spmm(rowptr, colind, val, B, 24, strat, seed=5, reduce=reduce)
    dB = oracle.spmm_backward(rowptr, colind, val, dC, 400, 24, strat, seed=5, reduce=reduce)
    lhs = float(np.sum(C.astype(np.float64) * dC))
    rhs = float(np.sum(B.astype(np.float64) * dB))
    assert abs(lhs - rhs) <= 1e-6 * abs(lhs)


@pytest.mark.parametrize("strat", [BUCKET, FASTRAND])
@pytest.mark.parametrize("reduce", [SUM, MEAN])
def test_backward_against_dense_brute_force(strat, reduce):
    rowptr, colind, val = synth.random_csr(70, 1300, seed=12, max_deg=40, special=(577, 1154, 600))
    dC = synth.dense(70, 6, seed=4)
    for s in (1, 5, 40, 2000):
        want = oracle.brute.spmm_backward(rowptr, colind, val, dC, 1300, s, strat, 7, reduce)
        got = oracle.spmm_backward(rowptr, colind, val, dC, 1300, s, strat, seed=7, reduce=reduce)
        assert _ulp_close(got, want, ulps=2)


def test_backward_ones_count_column_hits():
    """dC == 1, val == 1, SUM: dB[c, :] = number of sampled slots pointing at column c."""
    rowptr, colind, _ = synth.random_csr(300, 500, seed=1, max_deg=300, special=(577, 1154))
    for s in (1, 10, 1000):
        srp, sc, _, _ = oracle.sample(rowptr, colind, None, s, FASTRAND, seed=2)
        dB = oracle.spmm_backward(rowptr, colind, None, np.ones((300, 3), np.float32), 500, s,
                                  FASTRAND, seed=2)
        hits = np.bincount(sc, minlength=500).astype(np.float32)
        assert np.array_equal(dB, np.repeat(hits[:, None], 3, 1))


# ----------------------------------------------------------------- NEXT-4 variants
def test_prime_override_permutation_iff_coprime():
    """Generalisation of Eq. 2: j -> P' j mod d is a bijection of Z_d iff gcd(P', d) = 1."""
    for prime in (1, 2, 3, 7, 101, 577, 1009):
        for d in range(1, 260):
            ps = [oracle.position(FASTRAND, j, d, 0, prime) for j in range(d)]
            assert (sorted(ps) == list(range(d))) == (math.gcd(prime, d) == 1), (prime, d)
    # P' = 1 (and P' = 1 + d) is Bucket order
    assert [oracle.position(FASTRAND, j, 50, 0, 1) for j in range(50)] == list(range(50))
    assert [oracle.position(FASTRAND, j, 50, 0, 51) for j in range(50)] == list(range(50))


@pytest.mark.parametrize("prime", [2, 7, 1009])
def test_prime_override_against_brute_force(prime):
    rowptr, colind, val = synth.random_csr(60, 900, seed=3, max_deg=60, special=(14, 1009))
    B = synth.dense(900, 5, seed=1)
    for s in (1, 7, 100):
        want = oracle.brute.spmm(rowptr, colind, val, B, s, FASTRAND, 4, SUM, prime=prime)
        got = oracle.spmm(rowptr, colind, val, B, s, FASTRAND, seed=4, prime=prime)
        assert _ulp_close(got, want)
        srp, sc, _, spos = oracle.sample(rowptr, colind, val, s, FASTRAND, 4, prime=prime)
        d = np.diff(rowptr)
        for i in range(60):
            assert spos[srp[i]:srp[i + 1]].tolist() == oracle.brute.positions(FASTRAND, int(d[i]), s, 4, i, prime)


def test_mean_by_degree_variant():
    """MEAN by the original degree d_i (the other reading of L1571): with B == 1 every
    non-empty row is fp32(k_i)/fp32(d_i) exactly; brute force otherwise."""
    rowptr, colind, val = synth.random_csr(200, 800, seed=6, max_deg=150, special=(577,))
    d = np.diff(rowptr)
    ones = np.ones((800, 3), np.float32)
    for s in (1, 16, 1000):
        C = oracle.spmm(rowptr, colind, None, ones, s, FASTRAND, reduce=MEAN, mean_by_degree=True)
        k = np.minimum(d, s)
        want = np.where(d > 0, k.astype(np.float32) / np.maximum(d, 1).astype(np.float32), 0).astype(np.float32)
        assert np.array_equal(C, np.repeat(want[:, None], 3, 1))
        B = synth.dense(800, 4, seed=9)
        got = oracle.spmm(rowptr, colind, val, B, s, BUCKET, reduce=MEAN, mean_by_degree=True)
        exp = oracle.brute.spmm(rowptr, colind, val, B, s, BUCKET, 0, MEAN, mean_by_degree=True)
        assert _ulp_close(got, exp, ulps=2)
    # backward with the same divisor stays the adjoint
    B = synth.dense(800, 6, seed=2)
    dC = synth.dense(200, 6, seed=3)
    C = oracle.spmm(rowptr, colind, val, B, 12, FASTRAND, seed=1, reduce=MEAN, mean_by_degree=True)
    dB = oracle.spmm_backward(rowptr, colind, val, dC, 800, 12, FASTRAND, seed=1, reduce=MEAN,
                              mean_by_degree=True)
    assert abs(float(np.sum(C.astype(np.float64) * dC)) - float(np.sum(B.astype(np.float64) * dB))) \
        <= 1e-6 * abs(float(np.sum(C.astype(np.float64) * dC)))


# ---- the fp32 timing mode (bench.py's CPU baseline only; parity uses the fp64 oracle)
def test_f32_timing_mode_counts_and_bound():
    """oracle.spmm_f32: B = 1 and val = 1 give the sampled counts exactly (integers < 2^24), and
    with non-negative inputs it stays within the sequential fp32 sum bound gamma_k = k u / (1 - k u)
    of the fp64 oracle (+ one rounding for MEAN) -- a dropped slot, a wrong position or a
    mis-indexed B row fails one of them."""
    rowptr, colind, val = synth.random_csr(400, 900, seed=3, max_deg=300, special=(577, 1154))
    d = np.diff(rowptr)
    ones = np.ones((900, 24), np.float32)
    for strat in (BUCKET, FASTRAND):
        c = oracle.spmm_f32(rowptr, colind, None, ones, 64, strat, seed=0)
        assert np.array_equal(c, np.repeat(np.minimum(d, 64)[:, None], 24, 1).astype(np.float32))
        B = synth.dense(900, 40, seed=8)
        for s, red in ((16, SUM), (256, MEAN), (1000, SUM)):
            g = oracle.spmm_f32(rowptr, colind, val, B, s, strat, seed=0, reduce=red).astype(np.float64)
            o = oracle.spmm(rowptr, colind, val, B, s, strat, seed=0, reduce=red).astype(np.float64)
            mag = oracle.spmm(rowptr, colind, np.abs(val), np.abs(B), s, strat, seed=0, reduce=red).astype(np.float64)
            k = np.minimum(d, s).astype(np.float64)[:, None]
            u = 2.0 ** -24
            assert np.all(np.abs(g - o) <= (k * u / (1 - k * u) + 2 * u) * mag + 1e-30)
