"""Multi-GPU data paths run on ONE GPU with the real CUDA kernels (no injected oracle compute):

* B sharded by node blocks, all-gathered one 256-B feature slice at a time while the previous
  slice's slab pass runs (dist.BShardedSpMM) -- world 1, and 2 ranks sharing cuda:0 over gloo;
* the C all-gather fused into the epilogue over CUDA-IPC peer memory (dist.PeerBuffers), 2 ranks;
* the C all-gather through the NVLS multicast address of a torch symmetric-memory C
  (dist.MulticastC, multimem.st) -- world 1 (skipped where the node has no multicast support).

Every result is compared with the oracle (1e-5 bar) and, bitwise, with the single-GPU
replicated-B slab path (the multi-GPU C equals the 1-GPU C bitwise)."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_2104_10716_b200 as es  # noqa: E402
from paper_2104_10716_b200 import dist as esdist  # noqa: E402

N, NC, F, S = 903, 1100, 602, 96


def _graph():
    rowptr, colind, val = synth.random_csr(N, NC, seed=44, max_deg=300, special=(577, 1154))
    B = synth.dense(NC, F, seed=45, ld=608)
    return rowptr, colind, val, B


def _single_gpu_reference(rowptr, colind, val, B):
    dev = "cuda:0"
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ws = es.es_spmm_workspace(N, NC, len(colind), F, 608, S, True, device=dev, kernel="slab")
    return es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), S, 2, 7, 1, F=F, workspace=ws,
                             kernel="slab").cpu().numpy()


def _check(C, rowptr, colind, val, B):
    o = oracle.spmm(rowptr, colind, val, B, S, 2, seed=7, reduce=1, F=F)
    err = np.abs(C.astype(np.float64) - o)
    assert np.all(err <= np.maximum(1e-5 * np.abs(o), 1e-6)), err.max()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_bsharded(rank, world, dev, group=None):
    rowptr, colind, val, B = _graph()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    sh = esdist.plan(rowptr, S, F, world, rank)
    rp, ci, va = esdist.local_csr(rowptr, colind, val, sh)
    bs = esdist.BShardedSpMM(NC, F, world, rank, dev, group=group)
    b0, b1 = int(bs.blocks[rank]), int(bs.blocks[rank + 1])
    B_local = t(B[b0:b1, :F])                          # this rank's node block of B only
    ws = es.es_spmm_workspace(sh.r1 - sh.r0, NC, sh.e1 - sh.e0, 64, 64, S, True, device=dev, kernel="slab")
    C = torch.empty((sh.r1 - sh.r0, F), dtype=torch.float32, device=dev)
    bs(t(rp), t(ci), t(va), B_local, S, 2, 7, 1, C, n_rows=N, row_begin=sh.r0, row_end=sh.r1,
       nnz_base=sh.e0, nnz=sh.e1 - sh.e0, workspace=ws)
    torch.cuda.synchronize(dev)
    assert es.es_spmm_workspace_status(ws) == es.ES_WS_OK
    return sh, C.cpu().numpy()


def test_bsharded_pipelined_world1():
    rowptr, colind, val, B = _graph()
    _, C = _run_bsharded(0, 1, torch.device("cuda:0"))
    _check(C, rowptr, colind, val, B)
    assert np.array_equal(C, _single_gpu_reference(rowptr, colind, val, B))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda:0")                       # both ranks share the one GPU
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh, C_bs = _run_bsharded(rank, world, dev)
        rowptr, colind, val, B = _graph()
        peers = esdist.PeerBuffers(N, 608, device=dev)
        try:
            peers.C.fill_(-1.0)
            dist.barrier()
            full = esdist.sampled_spmm_fused_allgather(rowptr, colind, val, torch.from_numpy(B).to(dev), F, S, 2,
                                                       7, 1, peers)
            C_ag = full[:, :F].cpu().numpy()
            dist.barrier()
        finally:
            peers.close()
        q.put((rank, sh.r0, sh.r1, C_bs, C_ag))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rowptr, colind, val, B = _graph()
    ref = _single_gpu_reference(rowptr, colind, val, B)
    C_bs = np.concatenate([r[3] for r in res], axis=0)
    assert [r[1] for r in res] == [0, res[0][2]] and res[1][2] == N
    _check(C_bs, rowptr, colind, val, B)
    assert np.array_equal(C_bs, ref)                   # B-sharded pipelined == 1-GPU, bitwise
    for r in res:                                      # every rank holds the full C after the fused all-gather
        _check(r[4], rowptr, colind, val, B)


def test_multicast_allgather_world1():
    """The NVLS path on one rank: the multicast address of a 1-rank symmetric-memory C receives
    the epilogue's multimem.st stores (skipped where the node has no multicast support)."""
    port = _free_port()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda:0")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        try:
            mc = esdist.MulticastC(N, 608, device=dev)
        except Exception as exc:               # no NVLS on this node
            pytest.skip(f"no multicast: {exc}")
        rowptr, colind, val, B = _graph()
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        mc.C.fill_(-1.0)
        for kern in ("fused", "slab"):
            ws = es.es_spmm_workspace(N, NC, len(colind), F, 608, S, True, device=dev, kernel="slab") \
                if kern == "slab" else None
            es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), S, 2, 7, 1, F=F, C=mc.C, n_rows=N,
                              c_multicast=mc.multicast, workspace=ws, kernel=kern)
            torch.cuda.synchronize(dev)
            got = mc.C.cpu().numpy()
            _check(got[:, :F], rowptr, colind, val, B)
            assert np.all(got[:, F:] == -1.0)
    finally:
        dist.destroy_process_group()
