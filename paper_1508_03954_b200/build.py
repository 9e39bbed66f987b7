"""Builds libtreemg_b200.so in-tree with nvcc for sm_100a.

The library is the product: CUDA kernels + host C++ runner + the treemg
C-ABI (include/treemg.h, include/treemg_b200.h).  It is built into the
package directory so the .so travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtreemg_b200.so")
SOURCES = ["hierarchy.cu", "amr.cu", "fast.cu", "fused2.cu", "fused3.cu", "vcycles.cu", "dyn.cpp", "runner.cpp", "capi.cpp"]
HEADERS = ["hierarchy.hpp", "amr.hpp", "dyn.hpp", "exact_ops.cuh", "fast.cuh", "fused2.cuh", "fused3.cuh", "vcycles.cuh", "lattice.cuh", "runner.hpp",
           "slabs.inc"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS if os.path.exists(os.path.join(CSRC, f))]
    deps += [os.path.join(ROOT, "include", h) for h in ("treemg.h", "treemg_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = "", defines=()) -> str:
    """Compile libtreemg_b200.so for sm_100a (one nvcc per source file in
    parallel, then one link).  `out` / `defines` build a variant library
    elsewhere (developer A/B of compile-time parameters)."""
    import concurrent.futures as cf
    import tempfile
    target = out or LIB
    if not out and not force and not _stale():
        return LIB
    srcs = [os.path.join(CSRC, f) for f in SOURCES if os.path.exists(os.path.join(CSRC, f))]
    base = [nvcc_path()]
    # host compiler: the system g++ so libstdc++ is linked dynamically
    if os.path.exists("/usr/bin/g++"):
        base += ["-ccbin", "/usr/bin/g++"]
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
             "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-semantic-interposition", "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]
    flags += ["-D" + d for d in defines]
    tmp = tempfile.mkdtemp(prefix="tmg_build_")
    objs = [os.path.join(tmp, os.path.basename(src) + ".o") for src in srcs]

    def compile_one(i):
        return subprocess.run(base + flags + ["-c", srcs[i], "-o", objs[i]], capture_output=True, text=True, cwd=ROOT)

    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, range(len(srcs))))
    log = ""
    for src, res in zip(srcs, results):
        log += f"== {os.path.basename(src)}\n" + res.stdout + res.stderr
    link = base + ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xlinker", "-soname=libtreemg_b200.so",
                   "-o", target + ".tmp"] + objs
    ok = all(r.returncode == 0 for r in results)
    if ok:
        lres = subprocess.run(link, capture_output=True, text=True, cwd=ROOT)
        log += lres.stdout + lres.stderr
        ok = lres.returncode == 0
    if not out:
        with open(os.path.join(PKG, "build.log"), "w") as f:
            f.write(" ".join(base + flags) + "\n" + log)
    shutil.rmtree(tmp, ignore_errors=True)
    if not ok:
        raise RuntimeError("nvcc build failed:\n" + log[-6000:])
    os.replace(target + ".tmp", target)
    if verbose:
        print(log)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
