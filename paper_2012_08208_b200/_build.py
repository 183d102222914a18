"""Build libtopofilt.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtopofilt.so")
SOURCES = ["api.cu", "build.cu", "cl_build.cu", "dense_build.cu", "lattice_build.cu", "radix.cu", "scan.cu", "apply.cu", "stencil.cu", "oc.cu", "helmholtz.cu", "shard.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "topofilt.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile the library; `defines`/`out` build tuning variants (e.g. TF_APPLY_CW=8) elsewhere."""
    target = out or LIB
    if not defines and out is None and not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        obj = obj if not defines else obj.replace(".o", "_" + "_".join(d.replace("=", "") for d in defines) + ".o")
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = target + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                           "-o", tmp, "-lcudart"])
    os.replace(tmp, target)
    return target


def build_debug() -> str:
    """Variant with device-side bounds checks (TF_DCHECK -> __trap); load it with TOPOFILT_LIB."""
    return build(defines=("TF_DEBUG_CHECKS",), out=os.path.join(HERE, "..", "build_variants", "libtopofilt_debug.so"))


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv))
