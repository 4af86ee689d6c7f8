"""In-tree build of libimpm_gpu.so (sm_100a) with nvcc.

    python -m paper_2507_09435_b200.build
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "impm_sim.cu")
OUT = os.path.join(HERE, "libimpm_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-std=c++20", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-O3", "-shared",
]


def nccl_flags():
    """NCCL of the torch wheel (2.28; the same libnccl.so.2 torch.distributed
    loads, so one copy is mapped per process), else the system one."""
    try:
        import nvidia.nccl as nn
        root = list(nn.__path__)[0]
    except ImportError:
        root = None
    if root and os.path.exists(os.path.join(root, "include", "nccl.h")):
        lib = os.path.join(root, "lib")
        return ["-I" + os.path.join(root, "include"), "-L" + lib, "-l:libnccl.so.2",
                "-Xlinker", "-rpath=" + lib]
    return ["-lnccl"]


def sources():
    return [os.path.join(HERE, "csrc", f) for f in sorted(os.listdir(os.path.join(HERE, "csrc")))] + \
        [os.path.join(os.path.dirname(HERE), "include", "impm_gpu.h")]


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force=False, verbose=False, out=None):
    """out: another library path (A/B builds with IMPM_NVCC_EXTRA, loaded through IMPM_LIB)."""
    if out is None and not force and up_to_date():
        return OUT
    extra = os.environ.get("IMPM_NVCC_EXTRA", "").split()  # tuning experiments (e.g. -DIMPM_ASM_PPL3=2)
    cmd = [NVCC, *FLAGS, *extra, "-o", out or OUT, SRC, *nccl_flags()]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


REF_INCLUDE = "/root/reference/proj/include"
BAR_SWAP = os.path.join(os.path.dirname(HERE), "tests", "_build", "bar_swap")


def build_bar_swap(force=False):
    """tests/cpp/bar_swap.cpp: the reference's bar scenario with impm_gpu::MpmSim
    swapped in, compiled against the reference's own headers (only where
    /root/reference exists; the binary travels to the GPU box in-tree)."""
    src = os.path.join(os.path.dirname(HERE), "tests", "cpp", "bar_swap.cpp")
    hdr = os.path.join(os.path.dirname(HERE), "include", "impm_gpu.hpp")
    if not os.path.isdir(REF_INCLUDE):
        return BAR_SWAP if os.path.exists(BAR_SWAP) else None
    if not force and os.path.exists(BAR_SWAP) and all(
            os.path.getmtime(f) <= os.path.getmtime(BAR_SWAP) for f in (src, hdr, OUT)):
        return BAR_SWAP
    os.makedirs(os.path.dirname(BAR_SWAP), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(os.path.dirname(HERE), "include"),
                    "-I", REF_INCLUDE, "-o", BAR_SWAP, src, "-L", HERE, "-limpm_gpu",
                    "-Wl,-rpath,$ORIGIN/../../paper_2507_09435_b200"], check=True)
    return BAR_SWAP


if __name__ == "__main__":
    # python -m paper_2507_09435_b200.build [--force] [--out PATH]
    o = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    build(force="--force" in sys.argv, verbose=True, out=o)
