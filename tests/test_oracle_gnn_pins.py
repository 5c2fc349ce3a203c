"""Pins of the downstream GNN oracle (oracle/gnn.py::forward) against values fixed by hand,
not by another implementation of the same formulas.

Sources:
  * SPEC.md:L262-267 (gnn_layer examples): identity adjacency + identity weight -> h;
    ReLU([[-1, 2]]) = [[0, 2]]; 2-node path graph with self-loops, mean, identity weight,
    features [[2], [4]] -> [[3], [3]].
  * Eq. 1: H^{l+1} = sigma(A H^l W^l), GEMM first (GCN), bias after the
    aggregation, sigma between layers only (logits are the last layer's output).
  * GraphSage-mean, PAPER.md:L1256 / L1570-1575: h' = h W_self + mean_s(h) W_neigh + b.
Every expected value below is worked out by hand in the comment beside it, so a dropped term,
a swapped W_self / W_neigh, a ReLU on the last layer or a bias inside the aggregation fails."""
import numpy as np

import oracle
import oracle.gnn as ognn

B, F = oracle.BUCKET, oracle.FASTRAND


def csr(rows):
    rowptr = np.zeros(len(rows) + 1, np.int64)
    for i, r in enumerate(rows):
        rowptr[i + 1] = rowptr[i] + len(r)
    colind = np.array([c for r in rows for c in r], np.int32)
    return rowptr, colind


def layer(W, b=None, Wn=None):
    W = np.asarray(W, np.float32)
    out = {"W": W, "b": np.zeros(W.shape[1], np.float32) if b is None else np.asarray(b, np.float32)}
    if Wn is not None:
        out["W_neigh"] = np.asarray(Wn, np.float32)
    return out


def test_identity_gcn_is_h():
    # a = identity, weight = identity, activation none, sum -> output = h
    rp, ci = csr([[0], [1], [2]])
    h = np.array([[1.5, -2.0], [0.25, 3.0], [-7.0, 0.5]], np.float32)
    for strat in (B, F):
        out = ognn.forward("gcn", rp, ci, None, h, [layer(np.eye(2))], 4, strat)
        assert np.array_equal(out, h)


def test_relu_between_layers_not_after_the_last():
    # relu([[-1, 2]]) = [[0, 2]].  Two identity GCN layers on a self-loop graph:
    # layer 1 gives [[-1, 2]] -> ReLU -> [[0, 2]]; layer 2 (the logits) has no ReLU.
    rp, ci = csr([[0]])
    h = np.array([[-1.0, 2.0]], np.float32)
    two = ognn.forward("gcn", rp, ci, None, h, [layer(np.eye(2)), layer(np.eye(2))], 4, B)
    assert np.array_equal(two, [[0.0, 2.0]])
    # one layer = the last layer: no ReLU -> [[-1, 2]] stays negative
    one = ognn.forward("gcn", rp, ci, None, h, [layer(np.eye(2))], 4, B)
    assert np.array_equal(one, [[-1.0, 2.0]])
    # a negative last layer is kept: W = -I gives [[1, -2]] after the identity ReLU'd layer 1
    neg = ognn.forward("gcn", rp, ci, None, h, [layer(np.eye(2)), layer(-np.eye(2))], 4, B)
    assert np.array_equal(neg, [[0.0, -2.0]])


def test_path_graph_mean_is_3():
    # 2-node path graph with self-loops, mean aggregator, identity weight,
    # features [[2], [4]] -> [[3], [3]].  In the GraphSage form h W_self + mean(h) W_neigh + b
    # this is W_self = 0, W_neigh = I (the aggregation alone).
    rp, ci = csr([[0, 1], [0, 1]])
    h = np.array([[2.0], [4.0]], np.float32)
    for strat in (B, F):
        out = ognn.forward("sage", rp, ci, None, h, [layer([[0.0]], Wn=[[1.0]])], 8, strat)
        assert np.array_equal(out, [[3.0], [3.0]])
    # W_self = I, W_neigh = 0 -> h itself (pins which weight multiplies which term)
    out = ognn.forward("sage", rp, ci, None, h, [layer([[1.0]], Wn=[[0.0]])], 8, B)
    assert np.array_equal(out, h)
    # both: h + mean = [[5], [7]]
    out = ognn.forward("sage", rp, ci, None, h, [layer([[1.0]], Wn=[[1.0]])], 8, B)
    assert np.array_equal(out, [[5.0], [7.0]])


def test_gcn_bias_after_sum_aggregation():
    # Eq. 1 with bias: out = A (h W) + b.  Path graph with self-loops, SUM, W = [[2]], b = [1]:
    # hW = [[4], [8]]; A hW = [[12], [12]]; + b = [[13], [13]].  (Bias inside the aggregation,
    # A (hW + b), would give [[14], [14]].)
    rp, ci = csr([[0, 1], [0, 1]])
    h = np.array([[2.0], [4.0]], np.float32)
    out = ognn.forward("gcn", rp, ci, None, h, [layer([[2.0]], b=[1.0])], 8, B)
    assert np.array_equal(out, [[13.0], [13.0]])
    # weighted A (val carries the normalisation, reading R5): val = [0.5, 0.25 | 1, 1]
    val = np.array([0.5, 0.25, 1.0, 1.0], np.float32)
    out = ognn.forward("gcn", rp, ci, val, h, [layer([[2.0]], b=[1.0])], 8, B)
    # row 0: 0.5*4 + 0.25*8 + 1 = 5; row 1: 4 + 8 + 1 = 13
    assert np.array_equal(out, [[5.0], [13.0]])


def test_two_layer_graphsage_by_hand():
    # Graph (rows = neighbour lists): 0:{1,2}  1:{0}  2:{0,1,2}.  X (3x2):
    #   x0 = [1, 0], x1 = [0, 2], x2 = [2, 2]
    # Layer 1 (2 -> 2): W_self = [[1, 0], [0, 1]], W_neigh = [[0, 1], [1, 0]] (swap), b = [0, -1]
    #   mean: m0 = (x1 + x2)/2 = [1, 2]; m1 = x0 = [1, 0]; m2 = (x0+x1+x2)/3 = [1, 4/3]
    #   m W_neigh (swap): [2, 1], [0, 1], [4/3, 1]
    #   out = x + mW + b: h0 = [3, 0], h1 = [0, 2], h2 = [10/3, 2]   -> ReLU unchanged
    # Layer 2 (2 -> 1): W_self = [[1], [-1]], W_neigh = [[-1], [0]], b = [0.5]
    #   mean: m0 = (h1 + h2)/2 = [5/3, 2]; m1 = h0 = [3, 0]; m2 = (h0+h1+h2)/3 = [19/9, 4/3]
    #   h W_self: 3, -2, 4/3;  m W_neigh: -5/3, -3, -19/9
    #   logits: 3 - 5/3 + 0.5 = 11/6; -2 - 3 + 0.5 = -4.5; 4/3 - 19/9 + 0.5 = -5/18  (no ReLU)
    rp, ci = csr([[1, 2], [0], [0, 1, 2]])
    X = np.array([[1, 0], [0, 2], [2, 2]], np.float32)
    layers = [layer(np.eye(2), b=[0.0, -1.0], Wn=[[0, 1], [1, 0]]),
              layer([[1.0], [-1.0]], b=[0.5], Wn=[[-1.0], [0.0]])]
    out = ognn.forward("sage", rp, ci, None, X, layers, 8, B)
    want = np.array([[11 / 6], [-4.5], [-5 / 18]])
    assert np.allclose(out, want, rtol=0, atol=2e-6), out
    # s = 1 (Bucket keeps each row's first neighbour): m = [x1, x0, x0] in layer 1
    #   m W_neigh: [2, 0], [0, 1], [0, 1];  h0 = [3, -1] -> ReLU [3, 0]; h1 = [0, 2]; h2 = [2, 2]
    #   layer 2: m = [h1, h0, h0] = [0,2], [3,0], [3,0]; mW = 0, -3, -3
    #   logits: 3 - 0 + .5 = 3.5; -2 - 3 + .5 = -4.5; 0 - 3 + .5 = -2.5
    out1 = ognn.forward("sage", rp, ci, None, X, layers, 1, B)
    assert np.allclose(out1, [[3.5], [-4.5], [-2.5]], rtol=0, atol=1e-6), out1


def test_two_layer_gcn_by_hand():
    # Same graph, SUM over val = 1.  Layer 1 (2 -> 2): W = [[1, 1], [0, -1]], b = [0, 0]
    #   hW: x0 -> [1, 1]; x1 -> [0, -2]; x2 -> [2, 0]
    #   A hW: r0 = x1W + x2W = [2, -2]; r1 = x0W = [1, 1]; r2 = all three = [3, -1]
    #   ReLU: [2, 0], [1, 1], [3, 0]
    # Layer 2 (2 -> 1): W = [[1], [2]], b = [-1]
    #   hW: 2, 3, 3;  A hW: r0 = 3 + 3 = 6; r1 = 2; r2 = 2 + 3 + 3 = 8;  + b: 5, 1, 7
    rp, ci = csr([[1, 2], [0], [0, 1, 2]])
    X = np.array([[1, 0], [0, 2], [2, 2]], np.float32)
    layers = [layer([[1, 1], [0, -1]]), layer([[1.0], [2.0]], b=[-1.0])]
    for strat in (B, F):
        out = ognn.forward("gcn", rp, ci, None, X, layers, 8, strat)
        assert np.array_equal(out, [[5.0], [1.0], [7.0]])
