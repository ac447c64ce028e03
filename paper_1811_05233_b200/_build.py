"""Build libtorus.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with
the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import pathlib
import subprocess

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
SOURCES = [CSRC / "torus_abi.cu", CSRC / "torus_kernels.cu", CSRC / "torus_pull.cu",
           CSRC / "torus_nvls.cu"]
HEADERS = [CSRC / "torus_internal.h", CSRC / "torus_device.cuh", ROOT / "include" / "torus.h"]
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
        # one nvcc per translation unit, in parallel, then one link
        tmp = lib.with_name(f"{lib.name}.tmp{os.getpid()}")
        objs = [tmp.with_name(f"{p.stem}.{os.getpid()}.o") for p in SOURCES]
        compile_flags = [f for f in FLAGS if f not in ("-shared", "-cudart", "static")]
        procs = [subprocess.Popen([NVCC, *compile_flags, *[f"-D{d}" for d in defines], "-c", str(src),
                                   "-o", str(o)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                  text=True) for src, o in zip(SOURCES, objs)]
        logs = []
        failed = None
        for p in procs:
            out_s, err_s = p.communicate()
            logs.append(err_s)
            if p.returncode != 0:
                failed = (p.returncode, err_s)
        if failed is None:
            res = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                                  "-cudart", "static", *map(str, objs), "-o", str(tmp)],
                                 capture_output=True, text=True)
            if res.returncode != 0:
                failed = (res.returncode, res.stderr)
        for o in objs:
            if o.exists():
                o.unlink()
        if failed is not None:
            raise RuntimeError(f"nvcc failed ({failed[0]}):\n{failed[1][-4000:]}")
        log = "\n".join(logs)
        (PKG / "build_ptxas.log").write_text(log)
        if verbose:
            print(log)
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
