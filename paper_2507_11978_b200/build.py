"""Build libntb200.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels with the repo snapshot to the GPU box)."""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libntb200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I", str(PKG.parent / "include")]


def sources():
    return sorted(CSRC.glob("*.cu"))


def _digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
                    + [PKG.parent / "include" / "ntb200.h", Path(__file__)]):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: tuple = ()) -> Path:
    """Build libntb200.so; with ``variant`` build libntb200_<variant>.so with
    extra -D ``defines`` instead (tuning sweeps, selected by NTB_LIB_VARIANT)."""
    OUT_DIR.mkdir(exist_ok=True)
    lib = LIB if variant is None else OUT_DIR / f"libntb200_{variant}.so"
    stamp = OUT_DIR / (lib.stem + ".sha256")
    dig = _digest() + repr(defines)
    if lib.exists() and stamp.exists() and stamp.read_text() == dig and not force:
        return lib
    objs = []

    def compile_one(src: Path):
        obj = OUT_DIR / (src.stem + (f".{variant}" if variant else "") + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    cmd = [NVCC, *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart_static",
           "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    for o in objs:
        o.unlink(missing_ok=True)
    stamp.write_text(dig)
    return lib


if __name__ == "__main__":
    # python -m paper_2507_11978_b200.build [--force] [-v] [--variant TAG -DNAME=VAL ...]
    argv = sys.argv[1:]
    var = argv[argv.index("--variant") + 1] if "--variant" in argv else None
    defs = tuple(a[2:] for a in argv if a.startswith("-D"))
    print(build(force="--force" in argv, verbose="-v" in argv, variant=var, defines=defs))
