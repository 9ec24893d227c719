"""Build libdd.so in-tree: nvcc for the sm_100a kernels, g++ for the host
setup and C ABI, static cudart, NCCL from the torch-bundled wheel (the same
libnccl.so.2 torch loads, so one NCCL per process)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
SO = os.path.join(HERE, "libdd.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers (nvidia-nccl wheel) not found")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def build(force: bool = False, verbose: bool = False) -> str:
    nd = nccl_dir()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nd, "include")]
    os.makedirs(OBJ, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "dd.h")]
    newest = max(os.path.getmtime(d) for d in deps)
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= newest:
        return SO
    jobs = []
    for f in sources():
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJ, f + ".o")
        if f.endswith(".cu"):
            cmd = [os.path.join(CUDA, "bin", "nvcc"), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
                   *os.environ.get("DD_NVCC_DEFS", "").split(),
                   "--expt-relaxed-constexpr", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off",
                   *inc, "-c", src, "-o", obj]
        else:
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-Wall",
                   "-I", os.path.join(CUDA, "include"), *inc, "-c", src, "-o", obj]
        jobs.append(cmd)
    logs = []
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for out in ex.map(_run, jobs):
            logs.append(out)
    objs = [os.path.join(OBJ, f + ".o") for f in sources()]
    link = [os.path.join(CUDA, "bin", "nvcc"), *ARCH, "-shared", "-o", SO + ".tmp", *objs,
            "-cudart", "static", "-Xcompiler", "-fopenmp",
            "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    logs.append(_run(link))
    os.replace(SO + ".tmp", SO)
    with open(os.path.join(OBJ, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
