"""Autograd wrapper: the sampled SpMM as a differentiable op w.r.t. B (training variant).

PAPER.md §6.2 (L1577-1586) leaves training to future work: a fixed FastRand subset hurts
training accuracy, and DropEdge-style "different subset each iteration" sampling is what
training needs.  Here each call takes a `seed` (reading R6: seed != 0 rotates every row's
FastRand sequence), so passing the iteration number gives a new subset per iteration while
forward and backward of one iteration use the same subset.  Backward = es_spmm_backward
(dB = A_s^T dC).  The adjacency (rowptr, colind, val) is data, not a parameter.

With a `workspace` (es_spmm_workspace(...)), forward and backward take the feature-sliced path
and the backward reuses the slots the forward sampled into it (reuse_sampled), so each
iteration samples once.  The workspace must not be shared by two ops whose forward and
backward interleave.
"""
from __future__ import annotations

import torch

from . import ES_REDUCE_SUM, es_spmm_backward, es_spmm_backward_ex, es_spmm_run, es_spmm_run_ex


class SampledSpMM(torch.autograd.Function):
    @staticmethod
    def forward(ctx, B, rowptr, colind, val, s, strategy, seed, reduce, workspace):
        if workspace is None:
            C = es_spmm_run(rowptr, colind, val, B.contiguous(), s, strategy, seed, reduce)
        else:
            C = es_spmm_run_ex(rowptr, colind, val, B.contiguous(), s, strategy, seed, reduce,
                               F=B.shape[1], workspace=workspace)
        ctx.save_for_backward(rowptr, colind, val)
        ctx.cfg = (B.shape[0], B.shape[1], s, strategy, seed, reduce)
        ctx.workspace = workspace
        return C

    @staticmethod
    def backward(ctx, dC):
        rowptr, colind, val = ctx.saved_tensors
        n_cols, F, s, strategy, seed, reduce = ctx.cfg
        if ctx.workspace is None:
            dB = es_spmm_backward(rowptr, colind, val, dC.contiguous(), n_cols, s, strategy, seed, reduce, F=F)
        else:
            dB = es_spmm_backward_ex(rowptr, colind, val, dC.contiguous(), n_cols, s, strategy, seed, reduce,
                                     F=F, workspace=ctx.workspace, reuse_sampled=True)
        return dB, None, None, None, None, None, None, None, None


def sampled_spmm(B, rowptr, colind, val, s: int, strategy: int, seed: int = 0, reduce: int = ES_REDUCE_SUM,
                 workspace=None):
    """C = reduce_{sampled j} val_j * B[col_j] with autograd support w.r.t. B."""
    return SampledSpMM.apply(B, rowptr, colind, val, s, strategy, seed, reduce, workspace)
