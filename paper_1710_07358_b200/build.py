"""Build the in-tree native libraries for sm_100a.

    python -m paper_1710_07358_b200.build [--force] [--tuning]

- paper_1710_07358_b200/libb200reduce.so   the product (C ABI: include/b200reduce.h)
- build/tuning/libb200reduce.so             --tuning only: the same ABI compiled with
                                            -DRD_TUNING (reads the RD_TUNE_* knobs and
                                            carries the alternative exact-sum shapes;
                                            measurement tools load it explicitly)
- inputs/libinputs_host.so, inputs/libinputs_device.so   seeded generators
- oracle/liboracle.so                       the CPU checker (test infrastructure;
                                            building it is not using it)
- tools/libprobe.so                         the HBM read-bandwidth probe (measurement
                                            tooling: bench.py's same-run read ceiling)
- tools/libcubref.so                        CUB DeviceReduce::Reduce (bench.py's library
                                            context row; never on the product path)
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libb200reduce.so")
TUNING_OBJ = os.path.join(ROOT, "build", "obj_tuning")
TUNING_LIB = os.path.join(ROOT, "build", "tuning", "libb200reduce.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia.nccl
    return list(nvidia.nccl.__path__)[0]


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(INCLUDE, "b200reduce.h")])


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _compile(src: str, force: bool, tuning: bool = False, defines=(), objdir=None) -> str:
    objdir = objdir or (TUNING_OBJ if tuning else OBJ)
    obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
    if force or _stale(obj, [src] + _deps()):
        cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               *(["-DRD_TUNING"] if tuning else []), *[f"-D{d}" for d in defines],
               "-Xptxas", "-v", "-I", INCLUDE, "-I", CSRC, "-I", os.path.join(nccl_dir(), "include"),
               "-c", src, "-o", obj + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(obj + ".ptxas.log", "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
        os.replace(obj + ".tmp", obj)
    return obj


def build_library(force: bool = False, tuning: bool = False, defines=(), out: str | None = None) -> str:
    """The product library; `tuning` or `defines` + `out`: a measurement build
    of the same sources (A/B of design alternatives, tools/ab_lib.py)."""
    lib = out or (TUNING_LIB if tuning else LIB)
    objdir = (os.path.join(os.path.dirname(lib), "obj") if out else (TUNING_OBJ if tuning else OBJ))
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, tuning, defines, objdir), srcs))
    if force or _stale(lib, objs):
        nd = nccl_dir()
        cmd = ["nvcc", *ARCH, "-shared", "-o", lib + ".tmp", *objs,
               "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={os.path.join(nd, 'lib')}"]
        subprocess.check_call(cmd)
        os.replace(lib + ".tmp", lib)
    return lib


def build_probe(force: bool = False) -> str:
    src = os.path.join(ROOT, "tools", "probe.cu")
    out = os.path.join(ROOT, "tools", "libprobe.so")
    if force or _stale(out, [src]):
        subprocess.check_call(["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                               src, "-o", out + ".tmp"])
        os.replace(out + ".tmp", out)
    return out


def build_cub_ref(force: bool = False) -> str:
    """tools/libcubref.so: CUB DeviceReduce::Reduce, bench.py's library context row."""
    src = os.path.join(ROOT, "tools", "cub_ref.cu")
    out = os.path.join(ROOT, "tools", "libcubref.so")
    if force or _stale(out, [src]):
        subprocess.check_call(["nvcc", *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                               src, "-o", out + ".tmp"])
        os.replace(out + ".tmp", out)
    return out


def build_all(force: bool = False) -> None:
    sys.path.insert(0, ROOT)
    import inputs
    import oracle
    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        futs = [ex.submit(build_library, force), ex.submit(inputs.build_device, force),
                ex.submit(inputs.build_host, force), ex.submit(oracle.build, force),
                ex.submit(build_probe, force), ex.submit(build_cub_ref, force)]
        for f in futs:
            f.result()


if __name__ == "__main__":
    if "--define" in sys.argv:     # A/B build: --define NAME[,NAME2] --out build/ab/x/libb200reduce.so
        d = sys.argv[sys.argv.index("--define") + 1]
        o = os.path.abspath(sys.argv[sys.argv.index("--out") + 1])
        print(build_library(force="--force" in sys.argv, defines=tuple(d.split(",")), out=o))
    elif "--tuning" in sys.argv:
        print(build_library(force="--force" in sys.argv, tuning=True))
    else:
        build_all(force="--force" in sys.argv)
        print(LIB)
