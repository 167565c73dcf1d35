"""Build libcdms.so in-tree (nvcc, sm_100a).  `python -m paper_2604_19723_b200.build`."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libcdms.so")
LIB_TIMING = os.path.join(HERE, "libcdms_timing.so")  # debug variant with -DCDMS_PHASE_TIMING
SOURCES = ["loglik.cu", "taylor.cu", "nbmma.cu", "birth.cu", "response.cu", "beliefs.cu", "step.cu", "pf.cu", "slam.cu", "slam_step.cu", "lse.cu", "sort.cu", "cdms.cpp"]
HEADERS = ["cdms_internal.h", "geometry.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc() -> str:
    for cand in [os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"]:
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "cdms.h"),
                                                                 os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, timing: bool = False, variant: str | None = None,
          defines: list[str] | None = None) -> str:
    """Build libcdms.so; timing=True builds the phase-timing debug library; variant=NAME with defines builds
    an experiment library libcdms_NAME.so (debug / A-B measurements only, never loaded by default)."""
    if variant:
        lib = os.path.join(HERE, f"libcdms_{variant}.so")
    else:
        lib = LIB_TIMING if timing else LIB
    if not force and not variant and not _stale(lib):
        return lib
    obj_dir = OBJ + ("_timing" if timing else "") + (f"_{variant}" if variant else "")
    os.makedirs(obj_dir, exist_ok=True)
    inc, libdir = nccl_dirs()
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", inc, "-I", os.path.join(ROOT, "include")]
    if timing:
        common.append("-DCDMS_PHASE_TIMING")
    common += [f"-D{d}" for d in (defines or [])]

    def compile_one(src: str) -> str:
        out = os.path.join(obj_dir, src + ".o")
        cmd = [nvcc()] + ARCH + common + ["-Xptxas", "-v" if verbose else "-O3", "-c",
                                          os.path.join(CSRC, src), "-o", out]
        if src.endswith(".cpp"):
            cmd = [nvcc(), "-x", "cu"] + ARCH + common + ["-c", os.path.join(CSRC, src), "-o", out]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return out

    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    link = [nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + [
        "-L", libdir, "-l:libnccl.so.2", f"-Xlinker=-rpath={libdir}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, timing="--timing" in args, variant=var, defines=defs))
