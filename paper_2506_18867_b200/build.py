"""Build libbsfem.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("BSF_LIB_PATH", os.path.join(HERE, "libbsfem.so"))
SOURCES = ["host.cpp", "halo.cpp", "generic.cu", "tile.cu", "core.cu", "frame.cu", "band.cu", "g3.cu", "ip.cu", "solve.cu",
           "chol.cu", "contact.cu", "api.cu"]
HEADERS = ["host.hpp", "dev.hpp", "fbw.cuh", "tile.hpp", "core.hpp", "frame.hpp", "ip.hpp", "solve.hpp", "g3.hpp",
           "chol.hpp", "contact.hpp", "../../include/bsfem.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-cudart", "static"] + os.environ.get("BSF_EXTRA_NVCC_FLAGS", "").split()


CHECKED_LIB = os.path.join(HERE, "libbsfem_checked.so")   # -DBSF_CHECKED (shared-memory poisoning)


def _stale(lib=LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, lib: str = LIB, extra=()) -> str:
    if not force and not _stale(lib):
        return lib
    if os.path.abspath(lib) == CHECKED_LIB and "-DBSF_CHECKED" not in extra:
        extra = list(extra) + ["-DBSF_CHECKED"]
    flags = FLAGS + list(extra)
    objdir = os.path.join(HERE, "build" + ("_" + os.path.basename(lib).replace(".so", "") if lib != os.path.join(
        HERE, "libbsfem.so") else ""))
    os.makedirs(objdir, exist_ok=True)
    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *ARCH, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd = [NVCC, *ARCH, *flags, "-x", "c++", "-c", os.path.join(CSRC, src), "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    from concurrent.futures import ThreadPoolExecutor
    objs = []
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        for src, obj, r in ex.map(compile_one, SOURCES):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl", "-lpthread", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


def build_checked(force: bool = False) -> str:
    """The checked variant (-DBSF_CHECKED): every kernel poisons its shared memory with NaN first."""
    return build(force=force, lib=CHECKED_LIB, extra=["-DBSF_CHECKED"])


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
