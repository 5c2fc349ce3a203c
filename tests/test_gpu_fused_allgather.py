"""NEXT-1: the C all-gather fused into the SpMM epilogue (stores of every output row into every
rank's full C through peer pointers).  On one GPU: (1) two local buffers standing in for two
ranks' C, every row block stored into both; (2) two processes sharing cuda:0, peer buffers
mapped with CUDA IPC and handles exchanged over gloo -- the full multi-rank flow except the
NVLink transport itself."""
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

import paper_2104_10716_b200 as es  # noqa: E402
from paper_2104_10716_b200 import dist as esdist  # noqa: E402

N, NC, F = 900, 1200, 130


def graph(F=F):
    rowptr, colind, val = synth.random_csr(N, NC, seed=12, max_deg=200, special=(577,))
    B = synth.dense(NC, F, seed=4, ld=132)
    return rowptr, colind, val, B


@pytest.mark.parametrize("path", ["fused", "slab", "segstream"])
def test_two_local_peer_buffers(path):
    # slab: the feature-sliced path's epilogue stores to the peers too; segstream: the short-row
    # fused kernel's epilogue (F <= 128)
    with es.kernel_override(path):
        _two_local_peer_buffers(path, 128 if path == "segstream" else F)


def _two_local_peer_buffers(path, F):
    rowptr, colind, val, B = graph(F)
    dev = torch.device("cuda:0")
    bufs = [es.es_ipc_alloc(N * 132 * 4) for _ in range(2)]
    try:
        views = [torch.as_tensor(esdist._CudaArray(p, (N, 132)), device=dev) for p in bufs]
        for v in views:
            v.fill_(-1.0)
        peers = torch.tensor(bufs, dtype=torch.int64, device=dev)
        bounds = es.es_partition_rows(rowptr, 64, F, 3)
        Bd = torch.from_numpy(B).to(dev)
        for a, b in zip(bounds[:-1], bounds[1:]):
            e0, e1 = rowptr[a], rowptr[b]
            t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
            ws = (es.es_spmm_workspace(int(b - a), NC, int(e1 - e0), F, 132, 64, True, device=dev)
                  if path == "slab" else None)
            es.es_spmm_run_ex(t(rowptr[a:b + 1]), t(colind[e0:e1]), t(val[e0:e1]), Bd, 64, 2, 3, 1, F=F,
                              C=views[0], row_begin=int(a), row_end=int(b), n_rows=N, nnz_base=int(e0),
                              c_peers=peers, n_peers=2, workspace=ws, nnz=int(e1 - e0))
        torch.cuda.synchronize()
        want = oracle.spmm(rowptr, colind, val, B, 64, 2, seed=3, reduce=1, F=F)
        for v in views:
            got = v.cpu().numpy()
            assert np.allclose(got[:, :F], want, rtol=1e-5, atol=1e-6)
            assert np.all(got[:, F:] == -1.0)            # padding columns untouched
    finally:
        for p in bufs:
            es.es_ipc_free(p)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        rowptr, colind, val, B = graph()
        peers = esdist.PeerBuffers(N, 132, device=torch.device("cuda:0"))
        C = esdist.sampled_spmm_fused_allgather(rowptr, colind, val, torch.from_numpy(B).cuda(), F, 48, 2, 9, 0,
                                                peers, partition=es.es_partition_rows)
        q.put((rank, C[:, :F].cpu().numpy()))
        dist.barrier()
        peers.close()
    finally:
        dist.destroy_process_group()


def test_two_processes_ipc_fused_allgather():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rowptr, colind, val, B = graph()
    want = oracle.spmm(rowptr, colind, val, B, 48, 2, seed=9, reduce=0, F=F)
    for rank, C in res:
        assert np.allclose(C, want, rtol=1e-5, atol=1e-6), rank
