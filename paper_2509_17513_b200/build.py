"""Build libgsv_b200.so for sm_100a with nvcc (in-tree, no JIT cache).

Per-file flags: the fp64 translation units that must reproduce the
reference's rounding bit-for-bit (decode.cu: dequantization; project.cu:
projection and delta fold) are compiled with -fmad=false; everything else
may contract.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "lib"
LIB = OUT_DIR / "libgsv_b200.so"
OBJ_DIR = PKG / "lib" / "obj"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
               "--expt-relaxed-constexpr", "-Xcudafe", "--diag_suppress=177"] + ARCH
SOURCES = {
    "container.cpp": [],
    "decode.cu": ["-fmad=false"],
    "rc_decode.cu": [],
    "encode.cu": ["-fmad=false"],
    "project.cu": ["-fmad=false"],
    "sort.cu": [],
    "composite.cu": [],
    "render.cu": [],
    "api.cu": [],
}


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.h"), *CSRC.glob("*.cuh"), PKG.parent / "include" / "gsv_b200.h",
            Path(__file__)]
    t = obj.stat().st_mtime
    return any(d.exists() and d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    from concurrent.futures import ThreadPoolExecutor
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    objs = []
    relink = force or not LIB.exists()
    jobs = []
    for name, extra in SOURCES.items():
        src = CSRC / name
        obj = OBJ_DIR / (name + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            cmd = [nvcc(), "-c", str(src), "-o", str(obj), *NVCC_COMMON, *extra]
            if name.endswith(".cpp"):
                cmd = [nvcc(), "-x", "cu", "-c", str(src), "-o", str(obj), *NVCC_COMMON]
            jobs.append((name, cmd))
    # translation units compile in parallel (independent objects)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as pool:
        results = list(pool.map(lambda j: (j[0], subprocess.run(j[1], capture_output=True, text=True)), jobs))
    logs = []
    for name, r in results:
        logs.append((name, r.stdout + r.stderr))
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {name}")
        relink = True
    if relink:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), "-shared", *ARCH, "-o", str(tmp), *map(str, objs), "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, LIB)
    (OUT_DIR / "ptxas.log").write_text("".join(f"== {n}\n{l}\n" for n, l in logs)) if logs else None
    if verbose:
        for n, l in logs:
            print("==", n)
            print(l)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
