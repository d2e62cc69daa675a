"""Build libflashrnn.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2412_07752_b200.build [--verbose]

Every translation unit under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
``paper_2412_07752_b200/libflashrnn.so`` (git-ignored; it travels to the GPU
box with the gpurun snapshot).  Objects are cached under build/ by mtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", os.environ.get("FRNN_BUILD_TAG", "obj"))
LIB = os.environ.get("FRNN_BUILD_LIB", os.path.join(PKG, "libflashrnn.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
          "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"] + os.environ.get("FRNN_EXTRA_FLAGS", "").split()


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(ROOT, "include", "flashrnn.h"))
    hs.append(os.path.join(ROOT, "include", "flashrnn_dist.h"))
    return hs


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    newest_dep = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _headers()])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC] + ARCH + COMMON + ["-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    else:
        cmd += ["-x", "cu"]  # host C++ through nvcc so cuda headers/flags match
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcuda", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


TOOLS = ("frnn", "e2e_bench")  # tools/<name>.cpp -> build/<name>: C++ callers of the drop-in header


def build_tool(name: str) -> str:
    """g++ a tools/<name>.cpp program against include/ and libflashrnn.so."""
    exe = os.path.join(ROOT, "build", name)
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    cuda = os.path.dirname(os.path.dirname(NVCC))
    cmd = ["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(cuda, "include"),
           os.path.join(ROOT, "tools", name + ".cpp"), "-o", exe, "-L" + PKG, "-lflashrnn",
           "-L" + os.path.join(cuda, "lib64"), "-lcudart", "-lpthread",
           "-Wl,-rpath," + PKG + ":" + os.path.join(cuda, "lib64")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"g++ failed for tools/{name}.cpp:\n{r.stderr}")
    return exe


def build_tools() -> list:
    return [build_tool(n) for n in TOOLS]


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv))
