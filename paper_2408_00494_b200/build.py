"""In-tree build of libbssmppi.so (sm_100a) and the C oracle.

    python -m paper_2408_00494_b200.build
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libbssmppi.so"
LIB_EXACT = PKG / "libbssmppi_exact.so"   # libdevice transcendentals (A/B parity builds)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", *ARCH, "-Xcompiler", "-fPIC,-O2", "-shared",
              "-Xptxas", "-v", "-I", str(ROOT / "include")]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "bssmppi.h"]


def needs_build(target: Path, sources) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build_cuda(force: bool = False, verbose: bool = False, exact: bool = False) -> Path:
    target = LIB_EXACT if exact else LIB
    if force or needs_build(target, _sources()):
        defs = ["-DBSS_EXACT_MATH"] if exact else []
        cmd = [NVCC, *NVCC_FLAGS, *defs, str(CSRC / "bssmppi.cu"), "-o", str(target)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log = res.stdout + res.stderr
        (PKG / ("build_ptxas_exact.log" if exact else "build_ptxas.log")).write_text(log)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{log[-4000:]}")
        if verbose:
            print(log)
    return target


def build_oracle(force: bool = False) -> Path:
    """The C oracle (test infrastructure): oracle/Makefile."""
    res = subprocess.run(["make", "-C", str(ROOT / "oracle")] + (["-B"] if force else []),
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout}{res.stderr}")
    return ROOT / "oracle" / "liboracle.so"


if __name__ == "__main__":
    force = "-f" in sys.argv
    print(build_cuda(force, verbose="-v" in sys.argv))
    if "--exact" in sys.argv:
        print(build_cuda(force, exact=True))
    if (ROOT / "oracle" / "Makefile").exists():
        print(build_oracle(force))
