"""In-tree build of the sm_100a C-ABI library ``libhv_b200.so`` (nvcc + g++).

``python -m paper_2311_11425_b200.build`` or ``__graft_entry__.build()``.
The .so is written next to this file so it travels with the repo snapshot to
the GPU box (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
INCLUDE = HERE.parent / "include"
LIB = HERE / "libhv_b200.so"
OBJ = HERE / "csrc" / "_obj"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build the CUDA library")


def _sources():
    return sorted(CSRC.glob("*.cu")), sorted(CSRC.glob("*.cpp"))


def _digest(defines=()):
    h = hashlib.sha256()
    h.update(" ".join(defines).encode())
    for p in sorted(CSRC.glob("*")) + sorted(INCLUDE.glob("*.h")):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update(" ".join(ARCH).encode())
    return h.hexdigest()


def _run(cmd, verbose):
    if verbose:
        print(" ".join(str(c) for c in cmd), flush=True)
    r = subprocess.run([str(c) for c in cmd], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(map(str, cmd))}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr, file=sys.stderr)


def build(force=False, verbose=False, jobs=None, defines=(), lib=None):
    """Compile every CUDA/C++ source for sm_100a and link libhv_b200.so.

    ``defines``/``lib``: development builds (e.g. ``-DHV_PLANE_ABLATE`` into ablate/libhv_b200.so,
    loaded with HV_LIB=...) use their own object directory and never replace the product library.
    """
    lib_path = Path(lib) if lib else LIB
    obj_dir = OBJ if not defines else lib_path.parent / "_obj"
    stamp = lib_path.with_suffix(".sha256")
    dig = _digest(defines)
    if not force and lib_path.exists() and stamp.exists() and stamp.read_text().strip() == dig:
        return lib_path
    nvcc = _nvcc()
    obj_dir.mkdir(parents=True, exist_ok=True)
    cus, cpps = _sources()
    objs = []
    cmds = []
    for src in cus:
        obj = obj_dir / (src.stem + ".cu.o")
        cmds.append([nvcc, *ARCH, *defines, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp",
                     "-Xptxas", "-warn-spills", "-I", INCLUDE, "-c", src, "-o", obj])
        objs.append(obj)
    for src in cpps:
        obj = obj_dir / (src.stem + ".cpp.o")
        cmds.append(["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-I", INCLUDE,
                     "-I", "/usr/local/cuda/include", "-c", src, "-o", obj])
        objs.append(obj)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 2)) as ex:
        list(ex.map(lambda c: _run(c, verbose), cmds))
    tmp = lib_path.with_suffix(".so.tmp")
    _run([nvcc, *ARCH, "-shared", "-Xcompiler", "-fopenmp", "-o", tmp, *objs, "-lgomp"], verbose)
    os.replace(tmp, lib_path)
    stamp.write_text(dig)
    return lib_path


if __name__ == "__main__":
    if "--ablate" in sys.argv:   # development variants (HV_PLANE_VARIANT), tools/time_plane.py with HV_LIB
        print(build(force="--force" in sys.argv, verbose=True, defines=("-DHV_PLANE_ABLATE",),
                    lib=HERE.parent / "ablate" / "libhv_b200.so"))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
