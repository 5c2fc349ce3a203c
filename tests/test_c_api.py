"""The boundary is a real C ABI: the header compiles as C99 and C++, and a plain-C program
links against libesspmm.so (runs on a GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def test_header_compiles_as_c_and_cpp(tmp_path):
    src = tmp_path / "h.c"
    src.write_text('#include "es_spmm.h"\nint main(void){es_spmm_options_t o={0};(void)o;return ES_OK;}\n')
    for lang, std in (("c", "-std=c99"), ("c++", "-std=c++17")):
        subprocess.check_call(["gcc", "-x", lang, std, "-Wall", "-Werror", "-fsyntax-only", "-I",
                               os.path.join(ROOT, "include"), str(src)])


def _build_demo(out):
    from paper_2104_10716_b200 import _build
    _build.build()
    subprocess.check_call(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
                           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L",
                           os.path.join(ROOT, "paper_2104_10716_b200"), "-lesspmm", "-L", f"{CUDA}/lib64",
                           "-lcudart", "-lm", "-o", str(out)])


def test_c_demo_links(tmp_path):
    _build_demo(tmp_path / "demo")
    assert (tmp_path / "demo").exists()


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    exe = tmp_path / "demo"
    _build_demo(exe)
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2104_10716_b200") + ":" +
               os.environ.get("LD_LIBRARY_PATH", ""))
    res = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0/30 elements off" in res.stdout
    assert "0/432 off" in res.stdout                  # the slab path from C (workspace via options)
