"""Build libqal.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libqal.so")
SOURCES = ["qal_api.cu", "qal_magnus.cu", "qal_product.cu", "qal_grad.cu", "qal_dense.cu", "qal_blocks.cu", "qal_bigblocks.cu"]
HEADERS = ["qal_dev.cuh", "qal_slice.cuh", "qal_internal.h", "../../include/qal.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [*os.environ.get("QAL_NVCC_EXTRA", "").split(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


STAMP = os.path.join(HERE, "build", "flags.txt")


def _flags_text() -> str:
    """Everything that decides what libqal.so contains besides the sources: compiler and flag list
    (including QAL_NVCC_EXTRA experiment flags)."""
    return "\n".join([NVCC, *FLAGS, *SOURCES]) + "\n"


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    try:
        with open(STAMP) as f:
            if f.read() != _flags_text():   # built with other flags (e.g. an experiment build)
                return True
    except OSError:
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.getmtime(p) > t for p in deps)


def build_variant(name: str, extra: list) -> str:
    """Experiment build with extra nvcc flags into variants/libqal_<name>.so (never the in-tree
    libqal.so); load it with QAL_LIB=<path>."""
    out = os.path.join(HERE, "variants", f"libqal_{name}.so")
    objdir = os.path.join(HERE, "variants", f"build_{name}")
    return _compile(out, objdir, [*extra, *FLAGS], stamp=None)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    return _compile(OUT, os.path.join(HERE, "build"), FLAGS, stamp=STAMP, verbose=verbose)


def _compile(out_path: str, objdir: str, flags: list, stamp=None, verbose: bool = False) -> str:
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    logs = []
    for src, p in procs:
        out, _ = p.communicate()
        logs.append(f"== {src}\n{out}")
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed on {src}")
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    tmp = out_path + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, out_path)
    if stamp:
        with open(stamp, "w") as f:
            f.write(_flags_text())
    return out_path


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":   # _build.py --variant NAME FLAG...
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        build(force="--force" in sys.argv, verbose=True)
