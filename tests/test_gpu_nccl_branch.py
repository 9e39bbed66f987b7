"""The rank-per-process branch of the slab code (csrc/slabs.inc: ncclSend /
ncclRecv groups for the halo planes, the restriction partials and the level
L-2 gather; the norm gather of SlabGroup::cycle) executed on ONE GPU: the ranks
run as threads over tests/fake_nccl.cpp, a test double of the eight NCCL entry
points the library binds (loaded through TMG_NCCL_LIB in a fresh process, so
the product's one-time NCCL lookup sees it).  The double matches sends and
receives per (src, dst) pair in posting order like NCCL and rejects a pair
whose byte counts differ, so a wrong rank, offset or count in the exchange
lists fails here; the gathered iterate must be bitwise the single-GPU one."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_fake_nccl(outdir) -> str:
    sys.path.insert(0, ROOT)
    from paper_1508_03954_b200.build import nvcc_path
    lib = os.path.join(str(outdir), "libfake_nccl.so")
    cmd = [nvcc_path(), "-shared", "-std=c++17", "-Xcompiler", "-fPIC", "-Wno-deprecated-gpu-targets", "-o", lib,
           os.path.join(ROOT, "tests", "fake_nccl.cpp")]
    if os.path.exists("/usr/bin/g++"):
        cmd[1:1] = ["-ccbin", "/usr/bin/g++"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stdout + res.stderr
    return lib


def test_fake_nccl_builds_and_exports_the_bound_entry_points(tmp_path):
    """CPU: the double compiles, loads without a GPU and exports every NCCL
    symbol slabs.inc resolves (load_nccl); ids are distinct; a stray group end
    is refused."""
    import ctypes
    lib = ctypes.CDLL(build_fake_nccl(tmp_path))
    for sym in ("ncclGetUniqueId", "ncclCommInitRank", "ncclCommDestroy", "ncclSend", "ncclRecv", "ncclGroupStart",
                "ncclGroupEnd", "ncclGetErrorString", "fake_nccl_stats"):
        assert hasattr(lib, sym), sym
    a, b = ctypes.create_string_buffer(128), ctypes.create_string_buffer(128)
    assert lib.ncclGetUniqueId(a) == 0 and lib.ncclGetUniqueId(b) == 0
    assert a.raw != b.raw and a.raw.startswith(b"fake-nccl-")
    assert lib.ncclGroupEnd() != 0
    assert lib.ncclGroupStart() == 0 and lib.ncclGroupEnd() == 0


@pytest.mark.gpu
@pytest.mark.parametrize("levels,world,kind", [(4, 2, "td-add"), (4, 3, "td-bpx"), (5, 4, "td-add"), (5, 8, "td-bpx")])
def test_nccl_branch_ranks_bitwise_equal_single(tmp_path, levels, world, kind):
    lib = build_fake_nccl(tmp_path)
    env = dict(os.environ, TMG_NCCL_LIB=lib)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "nccl_ranks_worker.py"), str(levels), str(world),
                          kind, "5"], capture_output=True, text=True, env=env, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["ok"], out
    assert out["bitwise"], out
    assert out["same_across_ranks"], out
    assert out["norm_err"] <= 1e-13, out
    # per cycle and neighbour pair: 2 halo planes + 1 partial block (X1), 2 (X2), 2 or 4 (X3), the L-2 gather, norms
    assert out["sends"] >= 5 * (world - 1) * 7 and out["bytes"] > 0, out
