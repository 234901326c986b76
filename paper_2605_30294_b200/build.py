"""Build librafi.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2605_30294_b200.build [--force]

Compiles every CUDA/C++ source under csrc/ with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3``, links the CUDA
runtime statically and NCCL from the wheel torch itself loads (one NCCL per
process), and writes ``paper_2605_30294_b200/librafi.so``.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "librafi.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# proxy drivers: IEEE-exact float (no FMA contraction) so the CPU twins match bit for bit
PER_FILE = {"drivers.cu": ["-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false"]}


def nccl_paths():
    import nvidia.nccl  # torch's NCCL wheel (nvidia-nccl-cu12)

    base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(INCLUDE, "*")) + [__file__]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, defines=None, out: str | None = None) -> str:
    """Build librafi.so (or, with `defines`, a tuning variant at `out`)."""
    lib_path = out or LIB
    if not force and not defines and up_to_date():
        return LIB
    inc, libdir = nccl_paths()
    bdir = BUILD if not defines else os.path.join(BUILD, "v_" + os.path.basename(lib_path))
    os.makedirs(bdir, exist_ok=True)
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-Wall",
                     "-I", INCLUDE, "-I", inc, "-Xptxas", "-warn-spills"] + ["-D" + d for d in (defines or [])]
    if verbose:
        common += ["-Xptxas", "-v"]

    def compile_one(src):
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [NVCC] + common + PER_FILE.get(os.path.basename(src), []) + ["-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, "-x", "c++", "-std=c++17", "-O2", "-Xcompiler", "-fPIC,-Wall", "-I", INCLUDE, "-I", inc,
                   "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib_path + ".tmp.%d" % os.getpid()
    cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + [
        "-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath," + libdir]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    os.replace(tmp, lib_path)
    return lib_path


TOOLS = os.path.join(os.path.dirname(PKG), "tools")


def build_tools() -> list:
    """Measurement tools (not the product): tools/p2p_bw, the NVLink ceilings."""
    out = []
    for src in sorted(glob.glob(os.path.join(TOOLS, "*.cu"))):
        exe = src[:-3]
        if os.path.exists(exe) and os.path.getmtime(exe) >= os.path.getmtime(src):
            out.append(exe)
            continue
        r = subprocess.run([NVCC] + ARCH + ["-O3", "-lineinfo", "-o", exe, src], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
        out.append(exe)
    return out


VARIANTS = {  # scatter tuning experiments: name -> defines (build with --variants)
    "ilp2": ["RAFI_SCATTER_ILP=2"],
    "ilp8": ["RAFI_SCATTER_ILP=8"],
    "u4": ["RAFI_W_UNROLL=4"],
    "debug": ["RAFI_DEBUG_BOUNDS=1"],  # device-side bounds checks (scripts/sanitize_cases.py)
}


def build_variants(names=None):
    os.makedirs(os.path.join(PKG, "_variants"), exist_ok=True)
    return [build(force=True, defines=d, out=os.path.join(PKG, "_variants", "librafi_%s.so" % n))
            for n, d in VARIANTS.items() if not names or n in names]


if __name__ == "__main__":
    if "--variants" in sys.argv:
        i = sys.argv.index("--variants")
        names = sys.argv[i + 1].split(",") if i + 1 < len(sys.argv) and not sys.argv[i + 1].startswith("-") else None
        print(build_variants(names))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
