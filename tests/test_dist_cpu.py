"""World-size-2 gloo tests of the multi-GPU host logic on CPU (partition, slicing, B/C
all-gathers).  The per-rank compute is injected from the oracle -- the product default is
the CUDA library -- so these check the distribution logic, not the kernel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2104_10716_b200 import dist as esdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(sh, n_rows, rp, ci, va, B, F, s, strategy, seed, reduce):
    # rows [r0, r1) of the global CSR from the slice, seeded offsets by global id (row_base)
    rp_np = rp.numpy() - sh.e0
    return torch.from_numpy(oracle.spmm(rp_np, ci.numpy(), None if va is None else va.numpy(),
                                        B.numpy(), s, strategy, seed=seed, reduce=reduce, F=F,
                                        row_base=sh.r0))


def _partition(rowptr, s, F, world):
    import paper_2104_10716_b200 as es
    return es.es_partition_rows(rowptr, s, F, world)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rowptr, colind, val = synth.random_csr(611, 700, seed=5, max_deg=200, special=(577, 1154 // 2))
        F = 24
        B = synth.dense(700, F, seed=9)
        # replicated B, gather C
        C = esdist.sampled_spmm_distributed(rowptr, colind, val, torch.from_numpy(B), F, 40, 2, seed=13,
                                            reduce=1, gather_c=True, device="cpu",
                                            compute=_oracle_compute, partition=_partition)
        # sharded B (node blocks follow the same partition), gather C
        sh = esdist.plan(rowptr, 40, F, world, rank, partition=_partition)
        # B has 700 rows but the graph 611 rows: shard B by its own bounds over 700 rows
        rp_b = np.arange(701, dtype=np.int64)
        shb = esdist.plan(rp_b, 40, F, world, rank, partition=_partition)
        B_local = torch.from_numpy(B[shb.r0:shb.r1].copy())
        B_full = esdist.allgather_rows(B_local, shb.bounds)
        C2 = esdist.run_rows(sh, 611, *[torch.from_numpy(np.ascontiguousarray(x)) for x in
                                        esdist.local_csr(rowptr, colind, val, sh)],
                             B_full, F, 40, 2, 13, 1, compute=_oracle_compute)
        C2 = esdist.allgather_rows(C2, sh.bounds)
        q.put((rank, C.numpy(), C2.numpy(), B_full.numpy(), sh.bounds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_bitwise_equal_single(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rowptr, colind, val = synth.random_csr(611, 700, seed=5, max_deg=200, special=(577, 1154 // 2))
    B = synth.dense(700, 24, seed=9)
    want = oracle.spmm(rowptr, colind, val, B, 40, 2, seed=13, reduce=1)
    for rank, C, C2, B_full, bounds in res:
        assert bounds[0] == 0 and bounds[-1] == 611 and len(bounds) == world + 1
        assert np.array_equal(C, want)
        assert np.array_equal(C2, want)
        assert np.array_equal(B_full, B)


def test_plan_single_rank_is_everything():
    rowptr, colind, val = synth.random_csr(50, 60, seed=1)
    sh = esdist.plan(rowptr, 8, 16, 1, 0, partition=_partition)
    assert (sh.r0, sh.r1, sh.e0, sh.e1) == (0, 50, 0, int(rowptr[-1]))
    rp, ci, va = esdist.local_csr(rowptr, colind, val, sh)
    assert np.array_equal(rp, rowptr) and len(ci) == rowptr[-1]
