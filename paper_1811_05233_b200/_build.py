"""Build libtorus.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with
the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import pathlib
import subprocess

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
SOURCES = [CSRC / "torus_abi.cu", CSRC / "torus_kernels.cu", CSRC / "torus_pull.cu", CSRC / "torus_cast.cu",
           CSRC / "torus_baselines.cu", CSRC / "torus_ll.cu", CSRC / "torus_ll128.cu", CSRC / "torus_nvls.cu"]
HEADERS = [CSRC / "torus_internal.h", CSRC / "torus_device.cuh", CSRC / "torus_pull.h", CSRC / "torus_ll128.h",
           ROOT / "include" / "torus.h"]


def _deps(src: pathlib.Path, seen=None) -> set:
    """Headers a source includes (transitively, quoted includes only)."""
    import re
    seen = set() if seen is None else seen
    for m in re.finditer(r'#include "([^"]+)"', src.read_text()):
        h = (src.parent / m.group(1)).resolve()
        if h.exists() and h not in seen:
            seen.add(h)
            _deps(h, seen)
    return seen
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


def _dep_time(src: pathlib.Path) -> float:
    return max([src.stat().st_mtime] + [h.stat().st_mtime for h in _deps(src)])


def stale() -> bool:
    """The library is missing, older than a source or header, or linked from an object
    compiled before its source last changed (an edit made while nvcc was running)."""
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    if any(p.stat().st_mtime > t for p in SOURCES + HEADERS):
        return True
    odir = PKG / "build" / "default"
    return any(not (odir / f"{s.stem}.o").exists() or (odir / f"{s.stem}.o").stat().st_mtime < _dep_time(s)
               for s in SOURCES)


def build(force: bool = False, verbose: bool = False, out: pathlib.Path | None = None,
          defines: tuple[str, ...] = ()) -> pathlib.Path:
    """Compile each translation unit to an object (in parallel; objects are cached under
    build/ and reused while neither the source nor a header changed), then link."""
    lib = out or LIB
    if not (force or out is not None or stale()):
        return lib
    odir = PKG / "build" / ("default" if not defines else "_".join(defines).replace("=", "-"))
    odir.mkdir(parents=True, exist_ok=True)
    compile_flags = [f for f in FLAGS if f not in ("-shared", "-cudart", "static")]
    objs, procs = [], []
    for src in SOURCES:
        o = odir / f"{src.stem}.o"
        objs.append(o)
        dep_t = _dep_time(src)
        if not force and o.exists() and o.stat().st_mtime >= dep_t:
            continue
        tmp_o = o.with_name(f"{o.name}.tmp{os.getpid()}")
        procs.append((src, tmp_o, o, dep_t, subprocess.Popen(
            [NVCC, *compile_flags, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(tmp_o)],
            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    failed = None
    for src, tmp_o, o, dep_t, p in procs:
        _, err_s = p.communicate()
        (odir / f"{src.stem}.ptxas.log").write_text(err_s)
        if p.returncode != 0:
            failed = (p.returncode, err_s)
            if tmp_o.exists():
                tmp_o.unlink()
        else:
            os.replace(tmp_o, o)
            # stamp the object with the source time it was compiled from, so an edit
            # made while nvcc ran leaves it stale
            os.utime(o, (dep_t, dep_t))
    if failed is not None:
        raise RuntimeError(f"nvcc failed ({failed[0]}):\n{failed[1][-4000:]}")
    tmp = lib.with_name(f"{lib.name}.tmp{os.getpid()}")
    res = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                          "-cudart", "static", *map(str, objs), "-o", str(tmp)],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({res.returncode}):\n{res.stderr[-4000:]}")
    log = "\n".join((odir / f"{s.stem}.ptxas.log").read_text() for s in SOURCES
                     if (odir / f"{s.stem}.ptxas.log").exists())
    (PKG / "build_ptxas.log").write_text(log)
    if verbose:
        print(log)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
