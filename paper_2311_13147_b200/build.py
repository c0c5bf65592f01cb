"""Build libcyclicot.so in-tree with nvcc for sm_100a (B200). No torch in the library."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcyclicot.so")
SOURCES = ["abi.cu", "k_aggregate.cu", "k_expand.cu", "k_iter.cu", "k_iter_tma.cu", "k_iter_res.cu", "k_plan.cu", "k_shard.cu", "k_batch_cluster.cu", "k_batch_chain.cu", "k_srot.cu", "k_full.cu", "netsimplex.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
OBJDIR = os.path.join(HERE, "build_obj")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
LINK = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static"]


def _nccl_include() -> str:
    """Header of the NCCL torch loads (pip nvidia-nccl 2.28.x), not /usr/include's older copy. Only types and
    prototypes are used: the library dlopen()s libnccl.so.2 at run time."""
    try:
        import nvidia.nccl
        for base in nvidia.nccl.__path__:
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return "/usr/include"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "cyclicot.h"),
                                                                   __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    # one object per source, compiled in parallel, then one link (no relocatable device code)
    os.makedirs(OBJDIR, exist_ok=True)
    inc = _nccl_include()

    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] + [
        os.path.join(HERE, "..", "include", "cyclicot.h"), __file__]

    def compile_one(src):
        obj = os.path.join(OBJDIR, src + ".o")
        if not force and os.path.exists(obj) and all(
                os.path.getmtime(obj) > os.path.getmtime(p) for p in headers + [os.path.join(CSRC, src)]):
            return obj
        cmd = [NVCC, *FLAGS, "-I", inc, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    jobs = int(os.environ.get("COT_BUILD_JOBS", os.cpu_count() or 4))
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [NVCC, *LINK, "-o", LIB + ".tmp", *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
