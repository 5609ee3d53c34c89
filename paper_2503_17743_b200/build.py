"""Build libmoc3d.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Host C++ (laydown, ABI) is compiled with -ffp-contract=off and no fast-math
(App. A.7: host geometry must round the same way run to run); device code with
-fmad=false (no FMA contraction: the device fp64 OTF walk then rounds exactly as the
host walk and the oracle's -ffp-contract=off geometry; the fp32 physics uses explicit
fmaf, which is unaffected) and -lineinfo so ncu's source page maps to csrc/.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libmoc3d.so")
SOURCES = ["laydown.cpp", "partition.cpp", "capi.cpp", "solver.cu"]
HEADERS = ["host.h", "otf.h", "sweep_v2.cuh", "sweep_sc.cuh"]
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def _nccl_include() -> str:
    """nccl.h for types/prototypes (NCCL itself is dlopen'ed at run time): the pip
    nvidia-nccl headers matching torch's bundled libnccl.so.2, else the system ones."""
    try:
        import nvidia.nccl
        d = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    except ImportError:
        pass
    return "/usr/include"


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [
        os.path.join(HERE, "..", "include", "moc3d.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile libmoc3d.so (or a variant `out` with extra -D `defines`, for A/B runs)."""
    target = out or SO
    if out is None and not force and not _stale():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = target + ".tmp"
    cmd = [nvcc, ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-shared", "-o", tmp,
           "-I", _nccl_include()] + [f"-D{d}" for d in defines] + [
           "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-fno-fast-math",
           "-Xptxas", "-v" if verbose else "-O3",
           "-lgomp", "-ldl"] + [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=HERE)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("-")]
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = os.path.abspath(args[0]) if args else None
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=out, defines=defs))
