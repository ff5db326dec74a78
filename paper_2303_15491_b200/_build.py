"""In-tree build of the native libraries (no JIT cache: the built .so files
travel with the repository snapshot to the GPU box).

* ``libplmss_b200.so``  — the sm_100a CUDA kernels + C-ABI (include/plmss_b200.h).
* ``libplmss_dropin.so`` — the C++ facade implementing the reference's own
  ``plmss::`` entry points on top of the C-ABI (built only where the reference
  headers exist, i.e. in the build container; see csrc/dropin/).
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libplmss_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["capi.cu", "segment.cu", "combine.cu", "marching.cu", "scan.cu", "synth.cu", "fused.cu", "io.cu"]
NVCC_FLAGS = ARCH + [
    "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "--expt-relaxed-constexpr",
    "-I" + INCLUDE, "-I" + CSRC,
]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


LIB_CHECKED = os.path.join(PKG, "libplmss_b200_checked.so")


def build_cuda(force: bool = False, verbose: bool = False, checked: bool = False, variant: str = "",
               defines: tuple = ()) -> str:
    """checked=True: libplmss_b200_checked.so with the device bounds checks
    (-DPLMSS_CHECKED, fused.cu DCHECK), loaded when PLMSS_B200_LIB points at it.
    variant="x", defines=("-DFOO",): libplmss_b200_x.so, an A/B build of the same
    sources (same-box comparisons through PLMSS_B200_LIB)."""
    lib_path = LIB_CHECKED if checked else (os.path.join(PKG, f"libplmss_b200_{variant}.so") if variant else LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES]
    deps += [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    deps.append(os.path.join(INCLUDE, "plmss_b200.h"))
    if not force and not _stale(lib_path, deps):
        return lib_path
    objdir = os.path.join(PKG, "_obj_checked" if checked else (f"_obj_{variant}" if variant else "_obj"))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in SOURCES:
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC] + NVCC_FLAGS + (["-DPLMSS_CHECKED"] if checked else []) + list(defines) + \
            ["-c", os.path.join(CSRC, s), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd) + "\n" + out.decode())
        if verbose and out:
            print(out.decode())
    link = [NVCC] + ARCH + ["-shared", "-o", lib_path] + objs + ["-lcudart"]
    subprocess.run(link, check=True)
    return lib_path


DROPIN_DIR = os.path.join(CSRC, "dropin")


def build_dropin(force: bool = False):
    """C++ facade (plmss:: entry points over the C-ABI); needs the reference
    headers, so it is built only where /root/reference exists."""
    mk = os.path.join(DROPIN_DIR, "Makefile")
    if not os.path.exists(mk) or not os.path.isdir("/root/reference/proj/include"):
        return None
    subprocess.run(["make", "-s", "-j8", "-C", DROPIN_DIR] + (["-B"] if force else []), check=True)
    return os.path.join(ROOT, "build")


if __name__ == "__main__":
    import sys

    build_cuda(force="--force" in sys.argv, verbose=True)
    print(LIB)
