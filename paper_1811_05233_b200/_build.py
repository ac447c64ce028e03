"""Build libtorus.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with
the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import pathlib
import subprocess

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
SOURCES = [CSRC / "torus_abi.cu", CSRC / "torus_kernels.cu", CSRC / "torus_nvls.cu"]
HEADERS = [CSRC / "torus_internal.h", ROOT / "include" / "torus.h"]
LIB = PKG / "libtorus.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-shared", "-cudart", "static",
    "-Xptxas", "-v",
    f"-I{ROOT / 'include'}",
]


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: pathlib.Path | None = None,
          defines: tuple[str, ...] = ()) -> pathlib.Path:
    lib = out or LIB
    if force or out is not None or stale():
        tmp = lib.with_name(f"{lib.name}.tmp{os.getpid()}")
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], *map(str, SOURCES), "-o", str(tmp)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
        (PKG / "build_ptxas.log").write_text(res.stderr)
        if verbose:
            print(res.stderr)
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
