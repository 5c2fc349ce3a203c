#!/usr/bin/env python3
"""Benchmark of the ES-SpMM hot path (BASELINE.json metric) on 1..8 B200s.

One "step" = one pass of the whole hot path (degree/cap, sampling,
staging, gather-FMA, epilogue) over the configured graph, as ONE library call per rank on
the rank's row block: es_spmm_run_ex with a workspace when the library asks for one (the
feature-sliced path for B beyond L2: count + scan + sample materialisation + one slab kernel
per 64-float feature slice), else the single fused kernel (es_spmm_run_rows).  Inputs are
resident in HBM when the timed region starts; L2 is flushed (256 MiB write) before every
timed step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config reddit] [--F 602]
                  [--s 256] [--strategy fastrand|bucket] [--reduce mean|sum]
                  [--impl ours|reference]

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

FALLBACK_HBM_GBS = 6650.0      # /opt/skills/guides/B200_PROFILING.md fallback (only if no measured peak)
L2_RESIDENT_BYTES = 96 << 20   # a gathered operand up to this size stays L2-resident (126 MB L2; l2_peak.json)

DEFAULTS = {  # workload named in config.workload; BASELINE.json configs[3] (the graded target)
    "pubmed": dict(F=16, s=32, strategy="bucket", reduce="sum"),
    "arxiv": dict(F=128, s=64, strategy="fastrand", reduce="sum"),
    "proteins": dict(F=128, s=256, strategy="fastrand", reduce="sum"),
    "reddit": dict(F=602, s=256, strategy="fastrand", reduce="mean"),
    "scaled": dict(F=256, s=128, strategy="fastrand", reduce="sum"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="reddit", choices=sorted(DEFAULTS))
    ap.add_argument("--F", type=int, default=None)
    ap.add_argument("--s", type=int, default=None)
    ap.add_argument("--strategy", default=None, choices=["bucket", "fastrand"])
    ap.add_argument("--reduce", default=None, choices=["sum", "mean"])
    ap.add_argument("--seed", type=int, default=0, help="FastRand seed (0 = paper-exact Eq. 2)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto",
                    choices=["auto", "fused", "slab", "slab_smem", "slab_ldg", "slab_tma", "slab_stream", "tma", "warp",
                             "cpasync", "halfwarp", "rowstream", "grouped", "segstream"],
                    help="kernel family (A/B measurement through es_spmm_options_t.kernel; auto = the "
                         "library's plan, fused = never the feature-sliced path, slab* = that path wherever "
                         "it can run)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="warm-L2 variant (not the headline)")
    ap.add_argument("--allgather", action="store_true",
                    help="NEXT-1 variant: the C all-gather fused into the SpMM epilogue (every rank "
                         "stores its rows into all ranks' C over peer memory); N > 1")
    ap.add_argument("--allgather-mc", action="store_true",
                    help="the C all-gather fused into the epilogue through the NVLS multicast address of a "
                         "torch symmetric-memory C (multimem.st: one store per row reaches every rank)")
    ap.add_argument("--b-sharded", action="store_true",
                    help="B sharded by equal node blocks (the output of a previous layer): each step "
                         "all-gathers B one 256-B feature slice at a time on a side stream, overlapped with "
                         "the previous slice's slab pass (paper_2104_10716_b200.dist.BShardedSpMM)")
    ap.add_argument("--bf16", action="store_true",
                    help="NEXT-4 sensitivity variant: B stored as bf16 (fp32 accumulation); not the headline")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each step from a captured CUDA graph (auto: when a step < 0.5 ms, "
                         "i.e. launch-bound configs)")
    ap.add_argument("--cpu-seconds", type=float, default=3.0, help="wall-time target of the oracle sample")
    a = ap.parse_args()
    d = DEFAULTS[a.config]
    for k in ("F", "s", "strategy", "reduce"):
        if getattr(a, k) is None:
            setattr(a, k, d[k])
    if a.warmup < 3:
        a.warmup = 3
    return a


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def l2_peak():
    """The L2 streaming read rate measured on this pool's B200 (scripts/l2_peak.py ->
    profiles/l2_peak.json, with its clock record): the ceiling of L2-resident gathers."""
    path = os.path.join(ROOT, "profiles", "l2_peak.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return float(j["l2_stream_gbs"]), f"measured (profiles/l2_peak.json: {j['how'][:60]}..., {j.get('when')})"
    except Exception:
        return None, None


def ldb_for(F, elem=4):
    """B/C rows padded to a multiple of 32 B, the DRAM/L2 sector:
    F=602 fp32 -> 608 (2,432 B = 19 full 128-B L2 lines per gathered row)."""
    m = 32 // elem
    return (F + m - 1) // m * m


def workload_name(a):
    return (f"{a.config}-shaped synthetic CSR, F={a.F}, s={a.s}, {a.strategy}, "
            f"{'GraphSage mean' if a.reduce == 'mean' else 'GCN sum'}"
            + (", B stored bf16 (NEXT-4 variant)" if getattr(a, "bf16", False) else ""))


def byte_model(K, n_rows, F, b_elem=4):
    """Algorithmic bytes of one pass: 8K (sampled colind+val) + 8(N+1) (rowptr)
    + 4FK (B-row gathers; 2FK with bf16 storage) + 4FN (C store)."""
    return 8 * K + 8 * (n_rows + 1) + b_elem * F * K + 4 * F * n_rows


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.rows:
            return None
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 9:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------------ oracle timing (CPU baseline)
def oracle_sample_rows(rowptr, s, F, target_s, cores):
    """Every m-th row, m chosen so the fp64 oracle needs ~target_s wall seconds on `cores`."""
    d = np.diff(rowptr)
    k_all = int(np.minimum(d, s).sum())
    est_rate = 0.8e9 * cores            # slot*feature / s, rough; only sizes the sample
    m = max(1, int(np.ceil(k_all * F / (est_rate * target_s))))
    rows = np.arange(0, len(d), m, dtype=np.int64)
    return rows, m


def time_oracle(rowptr, colind, val, B, a, strat, red, rows):
    import oracle
    t0 = time.perf_counter()
    oracle.spmm(rowptr, colind, val, B, a.s, strat, seed=a.seed, reduce=red, F=a.F, rows=rows)
    return time.perf_counter() - t0


def cpu_baseline(rowptr, colind, val, B, a, strat, red, steps=1):
    """The oracle as it stands on the host cores (SURVEY 8(d) timing protocol): the fp64 parity
    oracle on every core (the reported value), plus the same sample in the fp32-FMA timing mode
    (a straightforward CPU port of Alg. 1) and the fp64 oracle on ONE core (a 1/cores sample)."""
    import oracle
    cores = oracle.max_threads()
    rows, m = oracle_sample_rows(rowptr, a.s, a.F, a.cpu_seconds, cores)
    d = np.diff(rowptr)
    Ks = int(np.minimum(d[rows], a.s).sum())
    ts = [time_oracle(rowptr, colind, val, B, a, strat, red, rows) for _ in range(steps)]
    t = float(np.median(ts))
    gf = lambda k, sec: 2.0 * a.F * k / sec / 1e9
    t0 = time.perf_counter()
    oracle.spmm_f32(rowptr, colind, val, B, a.s, strat, seed=a.seed, reduce=red, F=a.F, rows=rows)
    t32 = time.perf_counter() - t0
    rows1 = rows[::max(1, cores)]
    K1 = int(np.minimum(d[rows1], a.s).sum())
    oracle.set_threads(1)
    try:
        t1 = time_oracle(rowptr, colind, val, B, a, strat, red, rows1)
    finally:
        oracle.set_threads(cores)
    return {"value": gf(Ks, t), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"every {m}-th row of the same workload ({len(rows)} rows, {Ks} sampled edges), "
                      f"fp64 C oracle (oracle/es_oracle.c, -O2, OpenMP {cores} threads), "
                      f"median of {steps}, {t:.2f} s",
            "fp32_fma": {"value": round(gf(Ks, t32), 3), "cores": cores, "seconds": round(t32, 3),
                         "what": "the same sample, fp32 FMA accumulation in slot order (oracle.spmm_f32, "
                                 "timing mode only)"},
            "single_thread": {"value": round(gf(K1, t1), 3), "cores": 1, "seconds": round(t1, 3),
                              "sample": f"every {m * max(1, cores)}-th row ({len(rows1)} rows, {K1} sampled edges)"}}, t


# ------------------------------------------------------------------ main
def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    strat_id = 1 if a.strategy == "bucket" else 2
    red_id = 1 if a.reduce == "mean" else 0

    if a.impl == "reference":
        return main_reference(a, world, rank, strat_id, red_id)

    import torch
    import torch.distributed as dist
    import paper_2104_10716_b200 as es

    es.load_library()
    # one process per GPU; ES_BENCH_BACKEND=gloo lets a 1-GPU box exercise the multi-rank
    # flow (ranks then share cuda:0 -- validation only, never a reported scaling number)
    backend = os.environ.get("ES_BENCH_BACKEND", "nccl")
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1 or a.allgather_mc:               # symmetric memory needs a group, even of one rank
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    # ---------------- inputs (seeded, synthetic)
    rowptr, colind = synth.graph(a.config)
    n = len(rowptr) - 1
    nnz = int(rowptr[-1])
    F = a.F
    b_elem = 2 if a.bf16 else 4
    ldb = ldb_for(F, b_elem)
    _, seed_b = synth.seeds(a.config)
    B = synth.dense(n, F, seed_b, ld=ldb)
    val = np.ones(nnz, np.float32)                         # unweighted adjacency (L615), read by the kernel
    bounds = es.es_partition_rows(rowptr, a.s, F, world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    e0, e1 = int(rowptr[r0]), int(rowptr[r1])
    d_all = np.diff(rowptr)
    K_rank = int(np.minimum(d_all[r0:r1], a.s).sum())
    K_all = int(np.minimum(d_all, a.s).sum())

    rp_d = torch.from_numpy(rowptr[r0:r1 + 1].copy()).to(dev)
    ci_d = torch.from_numpy(colind[e0:e1]).to(dev)
    va_d = torch.from_numpy(val[e0:e1]).to(dev)
    B_d = torch.from_numpy(B).to(dev)                      # replicated: no collective on the timed path
    if a.bf16:
        B_d = B_d.to(torch.bfloat16)
    C_d = torch.empty((r1 - r0, ldb_for(F)), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    peers = mcast = bsh = None
    if a.allgather:
        from paper_2104_10716_b200.dist import PeerBuffers
        peers = PeerBuffers(n, C_d.stride(0), device=dev)
    if a.allgather_mc:
        from paper_2104_10716_b200.dist import MulticastC
        mcast = MulticastC(n, C_d.stride(0), device=dev)
    B_local = None
    if a.b_sharded:
        from paper_2104_10716_b200.dist import BShardedSpMM
        bsh = BShardedSpMM(n, F, world, rank, dev)
        b0, b1 = int(bsh.blocks[rank]), int(bsh.blocks[rank + 1])
        B_local = B_d[b0:b1].contiguous()
        del B_d                                            # this rank holds its block only
        B_d = B_local
    # the library's plan: a workspace (allocated once, outside the timed region) selects the
    # feature-sliced path when B does not fit L2 but a 64-float slab of it does
    slab_family = a.kernel in ("auto", "slab", "slab_smem", "slab_ldg", "slab_tma", "slab_stream")
    ws = (es.es_spmm_workspace(r1 - r0, n, e1 - e0, F, ldb, a.s, True, device=dev,
                               kernel=None if a.kernel == "auto" else a.kernel) if slab_family else None)
    if bsh is not None:                                    # one 64-float slice per call: force the slab path
        ws = es.es_spmm_workspace(r1 - r0, n, e1 - e0, 64, 64, a.s, True, device=dev, kernel="slab")
    kern = None if a.kernel == "auto" else a.kernel

    def launch(st, reuse=False):
        if bsh is not None:
            bsh(rp_d, ci_d, va_d, B_local, a.s, strat_id, a.seed, red_id, C_d, n_rows=n, row_begin=r0,
                row_end=r1, nnz_base=e0, nnz=e1 - e0, workspace=ws, stream=st)
        elif mcast is not None:
            es.es_spmm_run_ex(rp_d, ci_d, va_d, B_d, a.s, strat_id, a.seed, red_id, F=F, C=mcast.C,
                              row_begin=r0, row_end=r1, n_rows=n, nnz_base=e0, c_multicast=mcast.multicast,
                              workspace=ws, nnz=e1 - e0, kernel=kern, reuse_sampled=reuse, stream=st)
        elif peers is not None:
            es.es_spmm_run_ex(rp_d, ci_d, va_d, B_d, a.s, strat_id, a.seed, red_id, F=F, C=peers.C,
                              row_begin=r0, row_end=r1, n_rows=n, nnz_base=e0, c_peers=peers.peers,
                              n_peers=peers.world, workspace=ws, nnz=e1 - e0, kernel=kern, reuse_sampled=reuse,
                              stream=st)
        elif ws is not None or a.bf16 or kern is not None:
            es.es_spmm_run_ex(rp_d, ci_d, va_d, B_d, a.s, strat_id, a.seed, red_id, F=F, C=C_d,
                              row_begin=r0, row_end=r1, n_rows=n, nnz_base=e0, workspace=ws, nnz=e1 - e0,
                              kernel=kern, reuse_sampled=reuse, stream=st)
        else:                                  # the fused path, the rows' nnz stated (plan input)
            es.es_spmm_run_ex(rp_d, ci_d, va_d, B_d, a.s, strat_id, a.seed, red_id, F=F, C=C_d,
                              row_begin=r0, row_end=r1, n_rows=n, nnz_base=e0, nnz=e1 - e0, stream=st)

    lc0 = es.es_launch_count()
    for _ in range(a.warmup):
        if not a.no_flush:
            flush.zero_()
        launch(stream)
    torch.cuda.synchronize(dev)
    launches_per_step = (es.es_launch_count() - lc0) // a.warmup
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0.record(stream)
    launch(stream)
    w1.record(stream)
    torch.cuda.synchronize(dev)
    use_graph = a.graph == "on" or (a.graph == "auto" and w0.elapsed_time(w1) < 0.5)
    if use_graph:
        # the step's launches captured once and replayed: the timed region then holds the
        # kernel's device time instead of host launch latency (launch-bound small graphs)
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cap):
            launch(cap)
        stream.wait_stream(cap)
        torch.cuda.synchronize(dev)

        def step():
            graph.replay()
    else:
        def step():
            launch(stream)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.15)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    wall0 = time.perf_counter()
    for i in range(a.steps):
        if not a.no_flush:
            flush.zero_()                                  # evict L2 between timed steps
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    launches = launches_per_step * a.steps          # our kernels launched in the timed region
    clk = clocks.stop()

    per_step = np.array([s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]) / 1e3   # seconds
    t_rank = float(per_step.sum())
    t_max = t_rank
    if world > 1:
        tt = torch.tensor([t_rank], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    ms_per_step = 1e3 * t_max / a.steps
    flops_all = 2.0 * F * K_all                            # whole job per step (all ranks)
    value = flops_all / (t_max / a.steps) / 1e9            # GFLOP/s

    # ---------------- roofline of the dominant kernel, this rank's launches
    # Algorithmic bytes are SURVEY 8(d)'s per-run model, 8K + 8(N+1) + 4FK + 4FN, amortised over
    # the launches that do the gather-FMA.  The binding ceiling is the L2 streaming rate when the
    # gathered operand is L2-resident (the slab passes: one 256-B column slab of B at a time;
    # the fused kernels: B itself <= 96 MB), else HBM (profiles/l2_peak.json, MEASURED_PEAKS.json).
    hbm, hbm_src = measured_peaks()
    l2, l2_src = l2_peak()
    bytes_rank = byte_model(K_rank, r1 - r0, F, b_elem)
    avg_step = t_rank / a.steps
    step_achieved = bytes_rank / avg_step / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    key = f"{a.config}|F{F}|s{a.s}|{a.strategy}|{a.reduce}" + ("|slab" if ws is not None else "")
    if os.path.exists(prof) and world == 1:
        try:
            with open(prof) as f:
                tj = json.load(f)
            if key in tj:
                traffic = tj[key]["dram_bytes_per_launch"]
        except Exception:
            traffic = None
    bytes_model = ("8K + 8(N+1) + 2FK + 4FN (bf16 B)" if a.bf16 else
                   "8K + 8(N+1) + 4FK + 4FN (sampled colind+val, rowptr, B gathers, C)")
    if ws is None:
        # one fused launch per step: the step IS the dominant kernel's launch
        resident = n * ldb * b_elem <= L2_RESIDENT_BYTES
        t_launch = avg_step
        n_launch = 1
        kname = "es::spmm_cpasync<bf16>" if a.bf16 else es.es_spmm_plan(F, ldb, C_d.stride(0), B_d, C_d, s=a.s,
                                                                        n_rows=r1 - r0, nnz=e1 - e0)
        if a.kernel not in ("auto", "fused"):              # a forced family (A/B): not the plan's kernel
            kname = f"forced family '{a.kernel}' (es_spmm_options_t.kernel)"
        what = "one fused launch per step (sampling inside the kernel)"
    else:
        # slab path: the dominant kernel is the slab pass (one launch per 256-B feature slice,
        # ncu: ~97 % of the step).  Its launches are timed alone here, live, on the launch
        # stream with the same L2 flush: the same call with reuse_sampled=1 runs exactly the
        # slice passes over the slots the timed steps sampled into the workspace.
        lc = es.es_launch_count()
        launch(stream, reuse=True)                         # the slice passes alone: count them
        torch.cuda.synchronize(dev)
        n_launch = es.es_launch_count() - lc
        pe0 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
        pe1 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
        for i in range(a.steps):
            if not a.no_flush:
                flush.zero_()
            pe0[i].record(stream)
            launch(stream, reuse=True)
            pe1[i].record(stream)
        torch.cuda.synchronize(dev)
        t_launch = float(np.sum([x.elapsed_time(y) for x, y in zip(pe0, pe1)])) / 1e3 / a.steps   # s per step
        slab_row = -(-(F * b_elem) // (16 * n_launch)) * 16   # bytes of B per row and slice (widest)
        resident = n * slab_row <= L2_RESIDENT_BYTES       # one slab of B
        fam = a.kernel if a.kernel not in ("auto", "slab", "slab_flow") else \
            "es::spmm_slab_flow: persistent warps streaming slot-balanced row ranges"
        kname = f"slab pass ({fam}), one launch per feature slice ({n_launch}/step, <= {slab_row} B of each B row)"
        what = ("the slab passes alone (reuse_sampled), timed live; the step adds count + scan + sample "
                "materialisation")
    achieved = bytes_rank / t_launch / 1e9
    # the binding ceiling: the one the kernel runs closer to -- L2 (gathers served on chip) unless
    # the measured DRAM traffic (ncu, profiles/ncu_traffic.json) fills more of HBM than the
    # algorithmic bytes fill of the L2 rate; without a traffic record, by footprint
    dram_frac_live = (traffic / (t_launch / n_launch) / 1e9 / hbm) if (traffic and hbm) else None
    if l2 and dram_frac_live is not None:
        resident = achieved / l2 >= dram_frac_live
    bound, peak, src = ("l2", l2, l2_src) if (resident and l2) else ("hbm", hbm, hbm_src)
    roofline = {"bound": bound, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": src,
                "bytes_per_launch": int(bytes_rank / n_launch), "launches_per_step": n_launch,
                "launch_ms": round(1e3 * t_launch / n_launch, 4), "bytes_model": bytes_model + ", amortised over the "
                f"{n_launch} launch(es) of the gather-FMA", "kernel": kname, "what": what,
                "dram_frac": (round(traffic / (t_launch / n_launch) / 1e9 / hbm, 4) if traffic else None),
                "dram_traffic_source": f"profiles/ncu_traffic.json[{key}] (ncu dram__bytes_read+write per launch)"
                if traffic else None,
                "hbm_gather_model": {"achieved": round(achieved, 1), "peak": hbm, "frac": round(achieved / hbm, 4),
                                     "note": "the same algorithmic bytes against HBM: > 1 whenever the gathers "
                                             "are served by L2 -- not a roofline fraction"},
                "step": {"achieved": round(step_achieved, 1), "frac": round(step_achieved / peak, 4),
                         "launches": launches_per_step}}

    # ---------------- compulsory bytes: every B row the sample touches read once --
    # the distinct sampled columns come from our own sampler (es_spmm_sample), outside the timing
    compulsory = None
    if world == 1:
        _, s_col, _, _ = es.es_spmm_sample(rp_d, ci_d, None, a.s, strat_id, a.seed, row_base=r0, want_pos=False)
        n_touched = int(torch.unique(s_col).numel())
        del s_col
        compulsory = 8 * K_rank + 8 * (n + 1) + b_elem * F * n_touched + 4 * F * n

    # ---------------- end to end through the public host API (pinned host buffers)
    e2e = None
    if not a.no_e2e and not a.bf16:
        e2e = run_e2e(a, es, torch, dev, stream, rowptr, colind, val, B, r0, r1, e0, e1, F, ldb,
                      strat_id, red_id, flops_all, world, dist, backend)

    # ---------------- CPU baseline: the oracle as it stands, rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline and not a.bf16:
        cpu, _ = cpu_baseline(rowptr, colind, val, B, a, strat_id, red_id)

    if rank == 0:
        out = {
            "metric": f"sampled-SpMM GFLOP/s ({workload_name(a)})",
            "value": round(value, 2),
            "unit": "GFLOP/s",
            "n_gpus": world,
            "steps": a.steps,
            "warmup": a.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded; degree sequence fitted to PAPER.md Table dataset + Table sample_rate)",
            "config": {"workload": workload_name(a), "n_nodes": n, "nnz": nnz, "K_sampled": K_all,
                       "sampling_rate": round(K_all / nnz, 4), "F": F, "ldb": ldb, "s": a.s,
                       "strategy": a.strategy, "reduce": a.reduce, "seed": a.seed,
                       "l2": "no flush (warm)" if a.no_flush else "flushed between timed steps (256 MiB write)",
                       "parallelism": f"row-partitioned x{world} (sampled-byte balanced), "
                                      + ("B sharded by equal node blocks, all-gathered one 256-B feature slice at a "
                                         "time overlapped with the slab passes" if a.b_sharded else "B replicated")
                                      + ("; C all-gather fused into the SpMM epilogue (peer stores)"
                                         if a.allgather else "")
                                      + ("; C all-gather fused into the SpMM epilogue (NVLS multicast, multimem.st)"
                                         if a.allgather_mc else "")
                                      + ("" if backend == "nccl" else f" [{backend} validation run]"),
                       "timing": "sum of per-step CUDA-event times on the launch stream, max over ranks"
                                 + ("; each step replays a captured CUDA graph" if use_graph else "")},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches) * world,
            "clocks": clk,
            "detail": {"sampled_edges_per_s": K_all / (t_max / a.steps),
                       "input_edges_per_s": nnz / (t_max / a.steps),
                       "step_ms_min": round(1e3 * float(per_step.min()), 4),
                       "step_ms_median": round(1e3 * float(np.median(per_step)), 4),
                       "wall_s_timed_region": round(wall, 4),
                       "bytes_model_per_step_all_ranks": byte_model(K_all, n, F, b_elem),
                       "compulsory_bytes_per_step": compulsory,
                       "compulsory_model": "8K + 8(N+1) + 4F*N_touched + 4FN (each sampled B row read once; "
                                           "N_touched = distinct sampled columns, from es_spmm_sample)",
                       "ms_at_hbm_peak_for_compulsory_bytes": (round(1e3 * compulsory / (peak * 1e9), 4)
                                                               if compulsory else None)},
        }
        print(json.dumps(out), flush=True)
    if peers is not None:
        if world > 1:
            dist.barrier()                   # no rank unmaps while a peer may still write into it
        peers.close()
    if mcast is not None:
        mcast.barrier()
    if world > 1:
        dist.barrier()
    if dist.is_initialized():
        dist.destroy_process_group()


def run_e2e(a, es, torch, dev, stream, rowptr, colind, val, B, r0, r1, e0, e1, F, ldb, strat_id, red_id,
            flops_all, world, dist, backend):
    """Same metric through es_spmm_run_host: every step copies this rank's CSR slice and the
    replicated B from pinned host memory and reads C back (inside the timed region)."""
    rp_h = torch.from_numpy(rowptr[r0:r1 + 1].copy()).pin_memory()
    ci_h = torch.from_numpy(colind[e0:e1]).pin_memory()
    va_h = torch.from_numpy(val[e0:e1]).pin_memory()
    B_h = torch.from_numpy(B).pin_memory()
    # C's host rows at B's pitch (ldc = ldb): one linear device->host copy per chunk
    C_h = torch.empty((r1 - r0, ldb), dtype=torch.float32).pin_memory()
    need = es.es_spmm_host_workspace_bytes(r1 - r0, B.shape[0], e1 - e0, F, ldb, True)
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    pipe = es.HostPipeline()                                 # copy streams + events, created once
    steps = max(3, min(a.steps, 10))

    def one():
        es.es_spmm_run_host(rp_h, ci_h, va_h, B_h, a.s, strat_id, a.seed, red_id, F=F, C=C_h,
                            workspace=ws, row_base=r0, pipeline=pipe, stream=stream)

    for _ in range(2):
        one()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        one()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    t = ev0.elapsed_time(ev1) / 1e3
    pipe.close()
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    h2d = (rp_h.numel() * 8 + ci_h.numel() * 4 + va_h.numel() * 4 + B_h.numel() * 4)
    d2h = C_h.numel() * 4
    return {"value": round(flops_all / (t / steps) / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
            "ms_per_step": round(1e3 * t / steps, 3), "steps": steps,
            "api": "es_spmm_run_host_ex (pinned host buffers, chunked H2D/compute/D2H pipeline, the library's "
                   "plan on the device copies, copy streams reused across calls)"}


def main_reference(a, world, rank, strat_id, red_id):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only)."""
    if rank != 0:
        return 0
    import oracle
    rowptr, colind = synth.graph(a.config)
    n = len(rowptr) - 1
    F = a.F
    _, seed_b = synth.seeds(a.config)
    B = synth.dense(n, F, seed_b, ld=ldb_for(F))
    val = np.ones(len(colind), np.float32)
    cores = oracle.max_threads()
    target = max(0.5, a.cpu_seconds * 2.0 / max(1, a.steps + a.warmup) * 3)
    rows, m = oracle_sample_rows(rowptr, a.s, F, target, cores)
    d = np.diff(rowptr)
    Ks = int(np.minimum(d[rows], a.s).sum())
    for _ in range(a.warmup):
        time_oracle(rowptr, colind, val, B, a, strat_id, red_id, rows)
    ts = [time_oracle(rowptr, colind, val, B, a, strat_id, red_id, rows) for _ in range(a.steps)]
    t = float(np.sum(ts))
    value = 2.0 * F * Ks * a.steps / t / 1e9
    sample = (f"every {m}-th row of the same workload per step ({len(rows)} rows, {Ks} sampled edges), "
              f"fp64 C oracle, OpenMP {cores} threads")
    out = {"impl": "reference", "metric": f"sampled-SpMM GFLOP/s ({workload_name(a)})",
           "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": round(1e3 * t / a.steps, 3), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_name(a), "F": F, "s": a.s, "strategy": a.strategy,
                      "reduce": a.reduce},
           "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
