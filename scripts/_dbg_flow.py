import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
import paper_2104_10716_b200 as es
DEV = "cuda:0"
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
rowptr, colind, val = synth.random_csr(1301, 2300, seed=41, max_deg=400, special=(577, 1154, 1009, 300, 65, 33, 1))
B = synth.dense(2300, 128, seed=2)
d = np.diff(rowptr)
K = int(np.minimum(d, 256).sum())
lie = K // 2
nb = es.es_spmm_workspace_bytes(1301, 2300, lie, 128, 128, 256, True, kernel="slab")
ws = torch.zeros(nb, dtype=torch.uint8, device=DEV)
with es.kernel_override("slab"):
    C = es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 256, 2, 0, 1, F=128, workspace=ws, nnz=lie)
g = C.cpu().numpy()
bad = np.isnan(g).all(axis=1)
anyn = np.isnan(g).any(axis=1)
k = np.minimum(d, 256)
kp = (k + 3) // 4 * 4
srp = np.concatenate([[0], np.cumsum(kp)])
print("n", 1301, "K", K, "lie", lie, "Kpad", srp[-1], "bad rows", bad.sum(), "partial-nan rows", (anyn & ~bad).sum())
idx = np.nonzero(bad)[0]
print("first bad", idx[:20], "their k", k[idx[:20]], "srp end", srp[idx[:20] + 1])
print("last good", np.nonzero(~bad)[0][-5:])
o = oracle.spmm(rowptr, colind, val, B, 256, 2, reduce=1, F=128)
err = np.abs(g - o)
print("max err on good rows", np.nanmax(err[~bad]))
# normal call with a full workspace
ws2 = es.es_spmm_workspace(1301, 2300, len(colind), 128, 128, 256, True, device=DEV, kernel="slab")
with es.kernel_override("slab"):
    C2 = es.es_spmm_run_ex(t(rowptr), t(colind), t(val), t(B), 256, 2, 0, 1, F=128, workspace=ws2).cpu().numpy()
print("full ws: nan rows", np.isnan(C2).any(axis=1).sum(), "max rel err", float(np.max(np.abs(C2 - o) / np.maximum(np.abs(o), 1e-6))))
