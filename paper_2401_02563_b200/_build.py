"""In-tree build of the CUDA engine (libtgxd.so) for sm_100a.

The shared library is built next to this file so it travels with the repo
snapshot to the GPU box; there is no JIT cache and no CPU fallback.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libtgxd.so"
ROOT = PKG.parent

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC,-O3",
    "-shared",
    "-cudart", "static",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA engine cannot be built")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "tgxd.h"]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in sources())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(LIB), str(CSRC / "api.cu")]
    res = subprocess.run(cmd, cwd=str(PKG), capture_output=True, text=True)
    log = PKG / "build.log"
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    if verbose:
        print(res.stderr[-2000:])
    return LIB


def build_oracle(with_reference: bool | None = None) -> None:
    """Compile the test-side checkers (oracle/): the C restatement always, the
    reference library only where /root/reference exists (this container)."""
    targets = ["oracle"]
    if with_reference is None:
        with_reference = Path("/root/reference/proj/src").is_dir()
    if with_reference:
        targets.append("ref")
    res = subprocess.run(["make", "-C", str(ROOT / "oracle"), *targets],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout[-2000:]}\n{res.stderr[-4000:]}")


if __name__ == "__main__":
    print(build(force=True, verbose=True))
    build_oracle()
