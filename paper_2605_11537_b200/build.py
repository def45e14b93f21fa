"""Build the sm_100a C-ABI library ``libmoempmc.so`` in-tree with nvcc.

The library is the product: every hot-path kernel lives in ``csrc/`` behind
``include/moempmc.h``. It is compiled for ``sm_100a`` only (tcgen05/TMEM/TMA
do not exist on other targets), with the CUDA runtime linked statically so it
does not depend on which libcudart the host process (PyTorch) loaded.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libmoempmc.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-cudart", "static",
    "--expt-relaxed-constexpr",
]


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _fingerprint() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*")) + [INCLUDE / "moempmc.h"]):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None,
          out: Path | None = None) -> Path:
    """Compile csrc/*.cu into libmoempmc.so (skipped when sources are unchanged).

    ``extra``/``out``: diagnostic builds (e.g. ``-DMP_UNIT_TRACE`` into another file, used by
    tools/); the product library is always the plain build."""
    lib = Path(out) if out is not None else LIB
    extra = list(extra or [])
    stamp = lib.with_name("." + lib.stem + ".stamp")
    fp = _fingerprint() + " ".join(extra)
    if lib.exists() and stamp.exists() and stamp.read_text().strip() == fp and not force:
        return lib
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = ROOT / "build" / ("obj" if not extra else "obj_" + hashlib.sha256(" ".join(extra).encode()).hexdigest()[:8])
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    procs = []
    for src in _sources():
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra, f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((src, out.decode(errors="replace")))
        elif verbose and out:
            print(out.decode(errors="replace"), file=sys.stderr)
    if failed:
        msg = "\n".join(f"--- {s.name}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, *NVCC_FLAGS, "-shared", "-o", str(tmp), *map(str, objs), "-ldl", "-lpthread", "-lrt"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    stamp.write_text(fp + "\n")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
