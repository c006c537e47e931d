"""Build liblsk.so (sm_100a) in-tree with nvcc.
Usage: python paper_2006_07057_b200/build.py [-v] [--tuning]
(a script on purpose: importing the package would load a possibly stale liblsk.so).

--tuning builds scripts/variants/liblsk_tuning.so with -DLSK_TUNING: the measured alternatives
(warp-private and hybrid implicit kernels, pipelined team configurations) and the LSK_* tuning
environment knobs.  The product liblsk.so has neither (select a tuning build with
LSK_LIB_PATH)."""
from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "liblsk.so")
SOURCES = ["lsk_api.cu", "lsk_features.cu", "lsk_features_tc.cu", "lsk_sinkhorn.cu", "lsk_implicit.cu",
           "lsk_hybrid.cu", "lsk_grad.cu", "lsk_accel.cu", "lsk_resident.cu"]
TUNING_SOURCES = SOURCES + ["lsk_implicit_warp.cu", "lsk_implicit_tc.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore
        base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) \
            else list(nvidia.nccl.__path__)[0]
        inc = os.path.join(base, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    except Exception:
        pass
    return "/usr/include"


def _nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    return "nvcc"


def build(verbose: bool = False, ptxas_v: bool = False, tuning: bool = False) -> str:
    objdir = os.path.join(HERE, "build", "tuning") if tuning else os.path.join(HERE, "build")
    out = os.path.join(ROOT, "scripts", "variants", "liblsk_tuning.so") if tuning else OUT
    sources = TUNING_SOURCES if tuning else SOURCES
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-I" + os.path.join(ROOT, "include"), "-I" + nccl_include()]
    if tuning:
        common += ["-DLSK_TUNING"]
    if ptxas_v:
        common += ["-Xptxas", "-v"]

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        srcp = os.path.join(CSRC, src)
        deps = [srcp] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
        deps.append(os.path.join(ROOT, "include", "lsk.h"))
        if (not ptxas_v and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps)):
            return obj, ""
        cmd = [_nvcc(), "-c", srcp, "-o", obj] + common
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, res.stdout, res.stderr))
        return obj, res.stdout + res.stderr

    with concurrent.futures.ThreadPoolExecutor(len(sources)) as ex:
        results = list(ex.map(compile_one, sources))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log)
    tmp = out + ".%d.tmp" % os.getpid()   # renamed into place: a loaded copy stays valid
    link = [_nvcc(), "-shared", "-o", tmp] + objs + ARCH + ["-Xcompiler", "-fPIC", "-ldl"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n%s\n%s" % (res.stdout, res.stderr))
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(verbose=True, ptxas_v="-v" in sys.argv, tuning="--tuning" in sys.argv))
