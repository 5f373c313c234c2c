"""In-tree build of the sm_100a CUDA library (libnoma_b200.so) and the C++
host layer.  Compiles with nvcc directly -- no torch JIT, no site-packages
install -- so the built .so files travel to the GPU box with the snapshot."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libnoma_b200.so")
INCLUDE = os.path.join(ROOT, "include")

SOURCES = ["capi.cu", "k_lls.cu", "k_rng.cu", "k_train.cu", "k_train_w4.cu", "k_train_w8.cu", "k_train_w8d.cu", "k_train_l2.cu", "k_train_lat.cu", "k_train_f64.cu", "k_train_generic.cu", "k_dense.cu", "k_detect.cu", "k_detect_tc.cu"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(INCLUDE, "noma_cuda.h")]


def build(verbose: bool = False, ptxas_info: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cc = nvcc()
    hdrs = _headers()
    objs = []
    jobs = []
    # NOMA_BUILD_TRACE=1: the kernels with their cycle probes compiled in
    # (-DNOMA_PROBES: NOMA_PHASE_CLOCKS / NOMA_PHASE_TRACE / NOMA_LLS_CLOCKS /
    # NOMA_DETECT_CLK, tools/latency_probe.py); off in the product build
    trace = os.environ.get("NOMA_BUILD_TRACE") == "1"
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        tr = trace
        o = os.path.join(BUILD, src.replace(".cu", ".trace.o" if tr else ".o"))
        objs.append(o)
        if _stale(o, [s] + hdrs) or ptxas_info:
            cmd = [cc, *NVCC_FLAGS, *(["-DNOMA_PROBES"] if tr else []), "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o]
            if ptxas_info:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose or ptxas_info:
            sys.stderr.write(r.stdout + r.stderr)

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    stamp = os.path.join(BUILD, "link.txt")
    linked = open(stamp).read() if os.path.exists(stamp) else ""
    if _stale(LIB, objs) or linked != "\n".join(objs):
        cmd = [cc, "-shared", "-o", LIB, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
        with open(stamp, "w") as f:
            f.write("\n".join(objs))
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, ptxas_info="--ptxas" in sys.argv))
