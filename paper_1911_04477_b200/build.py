"""Build the sm_100a CUDA library in-tree: paper_1911_04477_b200/libbnn_b200.so.

Every .cu under csrc/ is compiled with nvcc for `-gencode arch=compute_100a,code=sm_100a`
(the B200 tcgen05/TMA feature set; nothing else is emitted) and linked into one shared
library whose exported symbols are the C ABI of include/bnn_cuda.h plus the C++
reference-signature API of include/bnn_b200.hpp (csrc/cpp_api.cpp, C++20). The .so is
git-ignored but travels to the GPU box with the repository snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libbnn_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
         f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


CXX = os.environ.get("CXX", "g++")
# the C++ reference-signature API (cpp_api.cpp) is C++20 like the reference (std::span)
# nlohmann/json (NetworkSpec JSON, csrc/io.cpp): the reference's own JSON library (network.cpp:6),
# used from the copy that ships inside the image's Python environment
JSON_INC = os.environ.get("BNN_JSON_INC", "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty")
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-fvisibility=hidden", "-Wall", f"-I{os.path.join(ROOT, 'include')}",
            "-I/usr/local/cuda/include", f"-I{JSON_INC}"]


def _compile(src: str) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "**", "*.h*"), recursive=True)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    if src.endswith(".cpp"):
        cmd = [CXX, *CXXFLAGS, "-c", src, "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB, *objs, "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(LIB)
    return LIB


CPP_TEST = os.path.join(PKG, "bin", "test_cpp_api")


def build_cpp_test(verbose: bool = False) -> str:
    """tests/cpp/test_cpp_api.cpp -> paper_1911_04477_b200/bin/test_cpp_api: the reference's unit
    cases through the C++ drop-in API, checked against the C oracle (test infrastructure)."""
    src = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
    orc = os.path.join(ROOT, "oracle", "_build")
    os.makedirs(os.path.dirname(CPP_TEST), exist_ok=True)
    cmd = [CXX, "-std=c++20", "-O1", "-Wall", f"-I{os.path.join(ROOT, 'include')}", src, "-o", CPP_TEST,
           f"-L{PKG}", "-lbnn_b200", f"-L{orc}", "-lbnn_oracle",
           "-Wl,-rpath,$ORIGIN/..", "-Wl,-rpath,$ORIGIN/../../oracle/_build"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ test build failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(CPP_TEST)
    return CPP_TEST


if __name__ == "__main__":
    build(verbose=True)
