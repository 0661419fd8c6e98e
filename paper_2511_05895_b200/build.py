"""Compile libdmf.so (sm_100a) in-tree with nvcc."""
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# DMF_LIB / DMF_EXTRA_NVCC select a diagnostic variant (e.g. -DDMF_DEBUG_BUSY into
# libdmf_debug.so); the product build is libdmf.so with the flags below.
LIB = os.environ.get("DMF_LIB") or os.path.join(PKG, "libdmf.so")
EXTRA = os.environ.get("DMF_EXTRA_NVCC", "").split()
SRC_DIR = os.path.join(PKG, "csrc")
SOURCES = [os.path.join(SRC_DIR, f) for f in ("dmf.cu",)]
DEPS = SOURCES + [os.path.join(SRC_DIR, f) for f in ("dmf_device.cuh", "solve.cuh")] + [os.path.join(ROOT, "include", "dmf.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = [NVCC, *FLAGS, *EXTRA, "-I", os.path.join(ROOT, "include"), "-o", LIB, *SOURCES]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stderr[-4000:])
        if verbose:
            print("\n".join(l for l in r.stderr.splitlines() if "k_solve" in l or "registers" in l)[-2000:])
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
