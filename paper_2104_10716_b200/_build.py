"""Build libesspmm.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["es_kernels.cu", "es_slab.cu", "es_backward_det.cu", "es_abi.cu"]
HEADERS = ["es_device.cuh", "es_internal.h"]
LIB = os.path.join(HERE, "libesspmm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--prec-div=true", "--prec-sqrt=true", "--fmad=true",   # never --use_fast_math (R8)
    "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "es_spmm.h"),
                                                                   __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def _check_no_spills(ptxas_log: str, src: str) -> None:
    """cp.async ring kernels that spill registers trapped with cudaErrorIllegalInstruction on
    B200 (profiles/r01.md); refuse to build one."""
    entry = None
    for line in ptxas_log.splitlines():
        if "Compiling entry function" in line:
            entry = line.split("'")[1] if "'" in line else line
        elif "spill stores" in line and entry and ("spmm_cpasync" in entry or "spmm_slab" in entry):
            stores = int(line.split("bytes spill stores")[0].split(",")[-1].strip().split()[0])
            if stores:
                raise RuntimeError(f"{src}: {entry} spills ({line.strip()}); lower its MINB")


def _check_sass(lib: str) -> None:
    """Reject a library whose SASS uses a 64-bit memory descriptor in an odd (misaligned)
    uniform register pair, e.g. `desc[UR1]`: ptxas 12.9 emitted that for a cache-hinted
    cp.async under register pressure and it traps (cudaErrorIllegalInstruction) on B200."""
    import re
    cuobjdump = os.path.join(os.path.dirname(NVCC), "cuobjdump")
    res = subprocess.run([cuobjdump, "-sass", lib], capture_output=True, text=True)
    if res.returncode != 0:
        return                                   # no disassembler: nothing to check
    fn = None
    bad = []
    for line in res.stdout.splitlines():
        if "Function : " in line:
            fn = line.split("Function : ")[1].strip()
        for m in re.finditer(r"desc\[UR(\d+)\]", line):
            if int(m.group(1)) % 2:
                bad.append((fn, line.strip()))
    if bad:
        raise RuntimeError("misaligned 64-bit uniform descriptor in SASS (illegal instruction on B200): "
                           + "; ".join(f"{f}: {l}" for f, l in bad[:3]))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
               "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(res.stderr)
        _check_no_spills(res.stderr, src)
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-lcudart_static", "-lrt", "-lpthread", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    _check_sass(tmp)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
