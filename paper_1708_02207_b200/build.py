"""In-tree build of libhdd_b200.so for sm_100a (nvcc, no JIT cache).

`python -m paper_1708_02207_b200.build` (or `__graft_entry__.build()`)
compiles csrc/*.cu + csrc/*.cpp into paper_1708_02207_b200/libhdd_b200.so.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libhdd_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = sources() + list(CSRC.glob("*.h")) + [ROOT / "include" / "hdd.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=()) -> Path:
    """Build libhdd_b200.so in-tree (or `out`, with extra -D `defines`, for A/B runs)."""
    target = Path(out) if out is not None else LIB
    if out is None and not force and not needs_build():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3", f"-I{ROOT / 'include'}", f"-I{CSRC}",
           *[f"-D{d}" for d in defines],
           *map(str, sources()), "-o", str(target) + ".tmp", "-lcudart"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed building libhdd_b200.so")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(str(target) + ".tmp", target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
