"""Build liblam.so (product) and synth/libsynth.so (input-generator harness) in-tree with nvcc for sm_100a.

No JIT cache: the .so files live next to their sources so they travel to the GPU box with the
repo snapshot.  Incremental by mtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIBLAM = os.path.join(PKG, "liblam.so")
LIBSYNTH = os.path.join(ROOT, "synth", "libsynth.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-Wall,-Wno-unused-function",
          "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)


def build(verbose: bool = False, force: bool = False) -> list[str]:
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "lam.h"))
    srcs = ["kernels.cu", "plan.cpp", "model.cpp", "control.cpp", "mcast.cpp", "runtime.cpp"]
    objs, jobs = [], []
    for s in srcs:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            lang = [] if s.endswith(".cu") else ["-x", "cu"]
            extra = ["-Xptxas", "-v"] if (verbose and s.endswith(".cu")) else []
            jobs.append([nvcc, *ARCH, *COMMON, *extra, *lang, "-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(_run, jobs))
    built = []
    if force or jobs or _stale(LIBLAM, objs):
        _run([nvcc, *ARCH, "-shared", "-o", LIBLAM, *objs, "-lrt", "-lpthread"])
        built.append(LIBLAM)
    ssrc = os.path.join(ROOT, "synth", "synth_gpu.cu")
    if force or _stale(LIBSYNTH, [ssrc, os.path.join(ROOT, "synth", "synth.cuh")]):
        _run([nvcc, *ARCH, *COMMON, "-shared", ssrc, "-o", LIBSYNTH])
        built.append(LIBSYNTH)
    return built


if __name__ == "__main__":
    import sys
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
