"""Build libwasabi.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libwasabi.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                 "-I", CSRC, "-Xptxas", "-warn-spills"] + os.environ.get("WASABI_NVCC_DEFS", "").split()
# the table kernels compute the fp32 rank keys with the specification's exact IEEE sequence
PER_FILE = {"kernels_tables.cu": ["--fmad=false"], "kernels_direct.cu": ["--fmad=false"],
            "kernels_coif.cu": ["--fmad=false"]}
SOURCES = ["kernels_tables.cu", "kernels_scan.cu", "kernels_bins.cu", "kernels_superpose.cu",
           "kernels_inverse.cu", "kernels_direct.cu", "kernels_coif.cu", "wasabi_host.cpp"]


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    deps = [src, os.path.join(CSRC, "internal.h"), os.path.join(CSRC, "device_common.cuh"),
            os.path.join(ROOT, "include", "wasabi.h")]
    return any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            cmd = [NVCC] + COMMON + PER_FILE.get(s, []) + ["-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
    if force or not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        tmp = OUT + f".{os.getpid()}.tmp"
        subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs)
        os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
