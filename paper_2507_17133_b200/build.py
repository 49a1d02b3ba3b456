"""Build libbrownout.so (sm_100a only) in-tree with nvcc.

    python -m paper_2507_17133_b200.build [--force]

Each csrc/*.cu is compiled to build/*.o (skipped when up to date), then linked
into paper_2507_17133_b200/libbrownout.so against the shared CUDA runtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "brownout")
LIB = os.path.join(PKG, "libbrownout.so")
# Instrumentation variant (python -m paper_2507_17133_b200.build --variant probe):
# -DBO_PROBE adds per-tile globaltimer stamps to the grouped GEMM (bo_probe_copy);
# loaded instead of the product library with BO_LIB=probe.  Never the default.
VARIANTS = {"probe": ["-DBO_PROBE"]}
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "--expt-relaxed-constexpr", "-I" + INCLUDE, "-I" + CSRC]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INCLUDE, "brownout.h"))
    return hs


def _compile(src: str, force: bool, verbose_ptxas: bool, variant: str | None = None) -> str:
    bdir = BUILD + ("_" + variant if variant else "")
    obj = os.path.join(bdir, os.path.basename(src)[:-3] + ".o")
    newest_dep = max(os.path.getmtime(p) for p in [src] + _headers())
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [nvcc()] + ARCH + CFLAGS + VARIANTS.get(variant, []) + (["-Xptxas", "-v"] if verbose_ptxas else []) + \
        ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose_ptxas:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose_ptxas: bool = False, variant: str | None = None) -> str:
    if variant is not None and variant not in VARIANTS:
        raise ValueError(f"unknown build variant {variant!r}")
    lib = LIB if variant is None else os.path.join(PKG, f"libbrownout_{variant}.so")
    os.makedirs(BUILD + ("_" + variant if variant else ""), exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose_ptxas, variant), srcs))
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        tmp = lib + ".tmp"
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "shared", "-o", tmp] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv, variant=var))
