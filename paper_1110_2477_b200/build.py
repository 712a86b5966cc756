"""Build libamtc.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libamtc.so")
SOURCES = ["amtc_capi.cu", "amtc_prepare.cu", "amtc_strip.cu", "amtc_light.cu", "amtc_full.cu", "amtc_crr.cu", "amtc_tree.cu"]
HEADERS = ["amtc_internal.cuh", "amtc_option.cuh", "pwl_device.cuh", "pwl_lane.cuh", "pwl_heavy.cuh", "amtc_root.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> str:
    """NCCL of the torch wheel (the same library torch.distributed loads)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        return list(spec.submodule_search_locations)[0]
    return "/usr"


NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(NCCL, "include")]
# developer experiments: extra nvcc flags (e.g. -DAMTC_LIGHT_CFG=6,6,8,3)
FLAGS += os.environ.get("AMTC_NVCC_EXTRA", "").split()
LINK = ["-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(NCCL, "lib")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "amtc.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = LIB + ".tmp"
    subprocess.run([NVCC, "-shared", *FLAGS, *objs, "-o", tmp, "-lcudart", *LINK], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
