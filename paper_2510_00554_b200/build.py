"""Build the in-tree native libraries with nvcc / gcc (no JIT cache).

* ``lib/libsentinel_b200.so`` -- the sm_100a kernels plus the C ABI declared
  in ``include/sentinel_b200.h``.
* ``_hostpack.so`` -- CPython helper (plain C) that packs sequences of host blocks / sample records
  into page-locked memory for the reference-shaped entry points (no hashing in it).
* ``oracle/_build/liboracle.so`` -- the plain-C CPU restatement used by the
  tests and by ``bench.py``'s CPU baseline (test infrastructure, never loaded
  by this package).
* ``tests/hostcheck/_build/libhostcheck.so`` -- host build of the kernels'
  per-thread code for the CPU suite.

nvcc cross-compiles without a GPU, so this runs in the build container; the
resulting ``.so`` files travel to the GPU box with the repository snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB_PATH = LIB_DIR / "libsentinel_b200.so"
HOSTPACK_LIB = PKG / "_hostpack.so"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "_build" / "liboracle.so"
HOSTCHECK_DIR = ROOT / "tests" / "hostcheck"
HOSTCHECK_LIB = HOSTCHECK_DIR / "_build" / "libhostcheck.so"
INTPEAK_BIN = ROOT / "tools" / "_build" / "intpeak"

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
]


def _nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found; cannot build libsentinel_b200.so")
    return exe


def _newer(target: Path, sources) -> bool:
    if not target.exists():
        return False
    t = target.stat().st_mtime
    return all(Path(s).stat().st_mtime <= t for s in sources)


def _run(cmd) -> None:
    proc = subprocess.run([str(c) for c in cmd], capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("build step failed: " + " ".join(str(c) for c in cmd))


def build_native(force: bool = False) -> Path:
    sources = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "sentinel_b200.h"]
    if not force and _newer(LIB_PATH, sources):
        return LIB_PATH
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    _run([_nvcc(), *NVCC_FLAGS, "-shared", *sorted(CSRC.glob("*.cu")), "-o", LIB_PATH])
    return LIB_PATH


def build_hostpack(force: bool = False) -> Path:
    import sysconfig
    src = CSRC / "hostpack.c"
    if not force and _newer(HOSTPACK_LIB, [src]):
        return HOSTPACK_LIB
    try:
        _run(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-pthread", "-Wall",
              "-I" + sysconfig.get_paths()["include"], src, "-o", HOSTPACK_LIB])
    except RuntimeError as exc:
        # the package runs without the helper (Python packers, same bytes); say so instead of failing the build
        sys.stderr.write(f"warning: _hostpack.so not built ({exc}); the reference-shaped calls pack in Python\n")
    return HOSTPACK_LIB


def build_oracle(force: bool = False) -> Path:
    src = ORACLE_DIR / "oracle.c"
    if not force and _newer(ORACLE_LIB, [src]):
        return ORACLE_LIB
    ORACLE_LIB.parent.mkdir(parents=True, exist_ok=True)
    _run(["gcc", "-O3", "-std=c11", "-fPIC", "-shared", "-pthread", src, "-o", ORACLE_LIB])
    return ORACLE_LIB


def build_hostcheck(force: bool = False) -> Path:
    sources = [HOSTCHECK_DIR / "hostcheck.cu"] + sorted(CSRC.glob("*.cuh"))
    if not force and _newer(HOSTCHECK_LIB, sources):
        return HOSTCHECK_LIB
    HOSTCHECK_LIB.parent.mkdir(parents=True, exist_ok=True)
    _run([_nvcc(), "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
          "-Xcompiler", "-fPIC", "-shared", HOSTCHECK_DIR / "hostcheck.cu", "-o", HOSTCHECK_LIB])
    return HOSTCHECK_LIB


def build_intpeak(force: bool = False) -> Path:
    src = ROOT / "tools" / "intpeak.cu"
    if not src.exists():
        return INTPEAK_BIN
    if not force and _newer(INTPEAK_BIN, [src]):
        return INTPEAK_BIN
    INTPEAK_BIN.parent.mkdir(parents=True, exist_ok=True)
    _run([_nvcc(), "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
          src, "-o", INTPEAK_BIN])
    return INTPEAK_BIN


REFERENCE_SRC = Path("/root/reference/pkg/src/sentinel")
REFERENCE_COPY = ORACLE_DIR / "_ref" / "sentinel"


def stage_reference(force: bool = False) -> Path:
    """Put the UNMODIFIED reference package where the GPU box can import it: ``oracle/_ref/sentinel``.

    The reference is pure Python, so "building" it is a copy of its package directory from the read-only
    tree it lives in. ``oracle/_ref/`` is git-ignored (no reference source enters the history) but travels
    with the snapshot, exactly like the built ``.so`` files. Only ``bench.py`` (the ``--impl reference`` arm
    and the ``cpu_baseline`` leg) and the tests import it, always as the thing measured against or checked
    with -- never by the product. Where ``/root/reference`` does not exist (the GPU box) this is a no-op
    and whatever travelled is used.
    """
    if not REFERENCE_SRC.is_dir():
        return REFERENCE_COPY
    newest = max(p.stat().st_mtime for p in REFERENCE_SRC.glob("*.py"))
    if not force and REFERENCE_COPY.is_dir() and all((REFERENCE_COPY / p.name).exists() for p in REFERENCE_SRC.glob("*.py")) \
            and min(p.stat().st_mtime for p in REFERENCE_COPY.glob("*.py")) >= newest:
        return REFERENCE_COPY
    if REFERENCE_COPY.exists():
        shutil.rmtree(REFERENCE_COPY)
    REFERENCE_COPY.parent.mkdir(parents=True, exist_ok=True)
    shutil.copytree(REFERENCE_SRC, REFERENCE_COPY, ignore=shutil.ignore_patterns("__pycache__"))
    return REFERENCE_COPY


def build_all(force: bool = False) -> None:
    build_native(force)
    build_hostpack(force)
    stage_reference(force)
    if (ORACLE_DIR / "oracle.c").exists():
        build_oracle(force)
    if (HOSTCHECK_DIR / "hostcheck.cu").exists():
        build_hostcheck(force)
    build_intpeak(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print(LIB_PATH)
