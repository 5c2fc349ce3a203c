"""Multi-GPU driver: 1-D row-block data parallelism over one node.

Every output row depends only on its own CSR row and on B (Alg. 1),
so the path shards into contiguous row blocks balanced by sampled bytes
(es_partition_rows, w_i = k_i(4F+8) + 4F).  Bounds are computed identically on every
rank from the host rowptr.  With B replicated there is no collective on the data path;
with B sharded by node blocks (the output of a previous layer) one all-gather of B
precedes the SpMM, and optionally one all-gather of C follows it (input of the next
layer).  Collectives go through torch.distributed (NCCL over NVLink 5 on B200; gloo in
the CPU tests).  The FastRand offset uses GLOBAL row ids and the per-row summation order
depends only on (k_i, F), so the gathered C is bitwise identical to a 1-GPU run.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Shard:
    rank: int
    world: int
    bounds: np.ndarray      # int64[world+1]
    r0: int                 # first global row of this rank
    r1: int                 # one past the last
    e0: int                 # first nonzero (absolute)
    e1: int


def plan(rowptr_host: np.ndarray, s: int, F: int, world: int, rank: int, partition=None) -> Shard:
    """Deterministic row blocks for `world` ranks (same on every rank)."""
    if partition is None:
        from . import es_partition_rows as partition
    bounds = np.asarray(partition(rowptr_host, s, F, world), dtype=np.int64)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    return Shard(rank, world, bounds, r0, r1, int(rowptr_host[r0]), int(rowptr_host[r1]))


def local_csr(rowptr_host, colind_host, val_host, sh: Shard):
    """This rank's CSR slice: rowptr entries stay ABSOLUTE (nnz_base = sh.e0)."""
    rp = np.ascontiguousarray(rowptr_host[sh.r0:sh.r1 + 1])
    ci = colind_host[sh.e0:sh.e1]
    va = None if val_host is None else val_host[sh.e0:sh.e1]
    return rp, ci, va


def allgather_rows(local, bounds: np.ndarray, group=None):
    """Concatenate per-rank row blocks (sizes from `bounds`) on every rank.
    Blocks are padded to the largest block for the equal-size all_gather_into_tensor."""
    import torch
    import torch.distributed as dist
    world = len(bounds) - 1
    sizes = np.diff(bounds)
    m = int(sizes.max()) if world else 0
    tail = tuple(local.shape[1:])
    buf = torch.zeros((m,) + tail, dtype=local.dtype, device=local.device)
    buf[: local.shape[0]].copy_(local)
    out = torch.empty((world * m,) + tail, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    parts = [out[r * m: r * m + int(sizes[r])] for r in range(world)]
    return torch.cat(parts, dim=0)


def run_rows(sh: Shard, n_rows: int, rp, ci, va, B, F: int, s: int, strategy: int, seed: int,
             reduce: int, C=None, stream=None, compute=None):
    """This rank's rows through the C ABI (es_spmm_run_rows).  `compute` lets CPU tests
    substitute a reference; the product default is the CUDA library (no fallback)."""
    if compute is not None:
        return compute(sh, n_rows, rp, ci, va, B, F, s, strategy, seed, reduce)
    from . import es_spmm_run_rows
    return es_spmm_run_rows(n_rows, rp, sh.e0, ci, va, B, s, strategy, seed, reduce, sh.r0, sh.r1,
                            F=F, C=C, stream=stream)


def sampled_spmm_distributed(rowptr_host, colind_host, val_host, B_local, F: int, s: int,
                             strategy: int, seed: int = 0, reduce: int = 0, *, b_sharded=False,
                             gather_c=False, group=None, device=None, compute=None, partition=None):
    """One distributed sampled SpMM.

    B_local: the full B (replicated) or, with b_sharded=True, this rank's node block
    B[bounds[r]:bounds[r+1]] (rows follow the same partition).  Returns this rank's C
    block, or the full C on every rank when gather_c=True."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n_rows = len(rowptr_host) - 1
    sh = plan(rowptr_host, s, F, world, rank, partition=partition)
    rp, ci, va = local_csr(rowptr_host, colind_host, val_host, sh)
    dev = device if device is not None else B_local.device

    def t(a):
        return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    B_full = allgather_rows(B_local, sh.bounds, group) if (b_sharded and world > 1) else B_local
    C = run_rows(sh, n_rows, t(rp), t(ci), t(va), B_full, F, s, strategy, seed, reduce,
                 compute=compute)
    if gather_c and world > 1:
        return allgather_rows(C, sh.bounds, group)
    return C


# --------------------------------------------------------------------------- B sharded, pipelined
def equal_blocks(n: int, world: int) -> np.ndarray:
    """Node blocks of B in the B-sharded mode: m = ceil(n / world) rows per rank (the last block
    shorter), so the all-gathered blocks ARE B's rows in order -- no compaction copy."""
    m = (n + world - 1) // world if world else n
    return np.minimum(np.arange(world + 1, dtype=np.int64) * m, n)


def _allgather_slab(out, send, group=None):
    """out (world*m x w) <- every rank's send (m x w), rank order.  NCCL on CUDA tensors; other
    backends (gloo: the multi-process validation on one GPU) stage through host memory."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        out[: send.shape[0]].copy_(send, non_blocking=True)
        return
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, send, group=group)
        return
    h_send = send.cpu()
    h_out = torch.empty(out.shape, dtype=out.dtype)
    dist.all_gather_into_tensor(h_out, h_send, group=group)
    out.copy_(h_out)


class BShardedSpMM:
    """One sampled SpMM with B SHARDED by node blocks (the output of a previous layer, SURVEY
    8(e)): C[:, c] needs only B[:, c] (Alg. 1 l.13-15), so the all-gather runs one 256-B feature
    slice at a time on a side stream and slice j+1's gather overlaps slice j's slab pass (the
    library's feature-sliced path over the gathered slab, double-buffered).  Exact: the same
    per-element order as the replicated-B slab path (bitwise).

    B_local: this rank's rows [blocks[r], blocks[r+1]) of B (equal_blocks), fp32, ldb columns.
    The call samples once (first slice) into the workspace and every other slice reuses it."""

    def __init__(self, n_cols: int, F: int, world: int, rank: int, device, group=None, width: int = 64):
        import torch
        self.n_cols, self.F, self.world, self.rank, self.group, self.w = n_cols, F, world, rank, group, width
        self.blocks = equal_blocks(n_cols, world)
        self.m = int(self.blocks[1] - self.blocks[0]) if world else n_cols
        self.slabs = [torch.empty((world * self.m, width), dtype=torch.float32, device=device) for _ in range(2)]
        self.send = [torch.empty((self.m, width), dtype=torch.float32, device=device) for _ in range(2)]
        self.comm = torch.cuda.Stream(device)
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]

    def __call__(self, rp, ci, va, B_local, s: int, strategy: int, seed: int, reduce: int, C, *, n_rows: int,
                 row_begin: int, row_end: int, nnz_base: int, nnz: int, workspace, stream=None):
        import torch
        from . import es_spmm_run_ex
        main = stream if stream is not None else torch.cuda.current_stream()
        n_sl = (self.F + self.w - 1) // self.w
        rows_here = B_local.shape[0]

        def gather(j):
            b = j % 2
            c0 = j * self.w
            w = min(self.w, self.F - c0)
            with torch.cuda.stream(self.comm):
                if j >= 2:
                    self.comm.wait_event(self.free[b])          # slab b consumed by slice j-2
                else:
                    self.comm.wait_stream(main)                 # B_local written before this call
                self.send[b][:rows_here, :w].copy_(B_local[:, c0:c0 + w])
                _allgather_slab(self.slabs[b], self.send[b], self.group)
                self.ready[b].record(self.comm)

        gather(0)
        for j in range(n_sl):
            if j + 1 < n_sl:
                gather(j + 1)                                   # overlaps slice j below
            b = j % 2
            c0 = j * self.w
            w = min(self.w, self.F - c0)
            main.wait_event(self.ready[b])
            es_spmm_run_ex(rp, ci, va, self.slabs[b], s, strategy, seed, reduce, F=w, C=C[:, c0:c0 + w],
                           row_begin=row_begin, row_end=row_end, n_rows=n_rows, nnz_base=nnz_base,
                           workspace=workspace, nnz=nnz, reuse_sampled=j > 0, stream=main)
            self.free[b].record(main)
        return C


# --------------------------------------------------------------------------- fused all-gather
class _CudaArray:
    """Minimal __cuda_array_interface__ holder to view a raw allocation as a torch tensor."""

    def __init__(self, ptr: int, shape: tuple):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class PeerBuffers:
    """A full-size C (n_rows x ldc fp32) on every rank, mapped into every other rank with CUDA
    IPC (es_ipc_*), for the SpMM whose epilogue writes each output row into all ranks' C over
    NVLink (the C all-gather fused into the SpMM, no separate collective).
    Handles are exchanged once with all_gather_object (any backend)."""

    def __init__(self, n_rows: int, ldc: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        from . import es_ipc_alloc, es_ipc_export, es_ipc_import
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n_rows, self.ldc = n_rows, ldc
        self.local_ptr = es_ipc_alloc(max(1, n_rows * ldc * 4))
        handles = [es_ipc_export(self.local_ptr)]
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, es_ipc_export(self.local_ptr), group=group)
        self.ptrs, self.imported = [], []
        for r, h in enumerate(handles):
            if r == self.rank:
                self.ptrs.append(self.local_ptr)
            else:
                ptr = es_ipc_import(h)
                self.ptrs.append(ptr)
                self.imported.append(ptr)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.peers = torch.tensor(self.ptrs, dtype=torch.int64, device=dev)
        self.C = torch.as_tensor(_CudaArray(self.local_ptr, (n_rows, ldc)), device=dev)

    def close(self):
        from . import es_ipc_close, es_ipc_free
        for ptr in self.imported:
            es_ipc_close(ptr)
        self.imported = []
        if self.local_ptr:
            es_ipc_free(self.local_ptr)
            self.local_ptr = 0


class MulticastC:
    """A full-size C (n_rows x ldc fp32) in torch symmetric memory on every rank of `group`, with
    the NVLS multicast address of the set: the SpMM epilogue stores each output
    row ONCE through it (es_spmm_options_t.c_multicast, multimem.st) and the NVSwitch delivers it
    to every rank -- 1x NVLink egress per row instead of (P-1)x unicast peer stores.  PyTorch does
    the plumbing (allocation, handle exchange, multicast binding); raises if the node has no
    multicast support (use PeerBuffers then)."""

    def __init__(self, n_rows: int, ldc: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        if not dist.is_initialized():
            raise RuntimeError("MulticastC needs an initialised process group (world size 1 included)")
        grp = group if group is not None else dist.group.WORLD
        if not symm._SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA, dev.index or 0):
            raise RuntimeError("no NVLS multicast support on this device (use PeerBuffers)")
        self.C = symm.empty((n_rows, ldc), dtype=torch.float32, device=dev)
        self.handle = symm.rendezvous(self.C, grp.group_name)
        if not self.handle.multicast_ptr:
            raise RuntimeError("no multicast address for this group (use PeerBuffers)")
        self.multicast = int(self.handle.multicast_ptr)
        self.world = self.handle.world_size
        self.rank = self.handle.rank

    def barrier(self):
        self.handle.barrier()


def sampled_spmm_fused_allgather(rowptr_host, colind_host, val_host, B, F: int, s: int, strategy: int,
                                 seed: int, reduce: int, peers: PeerBuffers, group=None, partition=None):
    """This rank's row block through es_spmm_run_ex with the fused all-gather epilogue; on
    return (after a barrier) peers.C holds the FULL C on every rank."""
    import torch
    import torch.distributed as dist
    from . import es_spmm_run_ex
    n_rows = len(rowptr_host) - 1
    sh = plan(rowptr_host, s, F, peers.world, peers.rank, partition=partition)
    rp, ci, va = local_csr(rowptr_host, colind_host, val_host, sh)
    dev = B.device

    def t(a):
        return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    es_spmm_run_ex(t(rp), t(ci), t(va), B, s, strategy, seed, reduce, F=F, C=peers.C,
                   row_begin=sh.r0, row_end=sh.r1, n_rows=n_rows, nnz_base=sh.e0,
                   c_peers=peers.peers, n_peers=peers.world)
    torch.cuda.synchronize(dev)
    if peers.world > 1:
        dist.barrier(group=group)
    return peers.C
