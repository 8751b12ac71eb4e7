"""Build libaxe.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.environ.get("AXE_BUILD_OUT") or os.path.join(HERE, "libaxe.so")  # dev A/B variants only
BUILD = os.path.join(ROOT, "build", "axe" + ("_" + os.path.basename(OUT) if os.environ.get("AXE_BUILD_OUT") else ""))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    for p in (spec.submodule_search_locations or []) if spec else []:
        if os.path.exists(os.path.join(p, "lib", "libnccl.so.2")):
            return p
    raise RuntimeError("pip NCCL (nvidia.nccl, the one torch loads) not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = (sources() + glob.glob(os.path.join(CSRC, "*.h*")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
            [os.path.join(ROOT, "include", "axe.h"), __file__])
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    nccl = nccl_dir()
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-Wall", "-I", os.path.join(ROOT, "include"),
              "-I", CSRC, "-I", os.path.join(nccl, "include")] + ARCH
    if os.environ.get("AXE_PTXAS_VERBOSE"):
        common += ["-Xptxas", "-v"]
    common += os.environ.get("AXE_EXTRA_NVCC", "").split()  # dev A/B variants only

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [NVCC] + common + ["-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, "-x", "cu"] + common + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [NVCC, "-shared"] + ARCH + os.environ.get("AXE_EXTRA_LINK", "").split() + ["-cudart", "static", "-o", tmp] + objs + [
        "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
