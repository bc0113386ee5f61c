"""Compile libpwb200.so in-tree for sm_100a (nvcc; no torch extension machinery).

K1 is specialised per vector dimension (compile-time pairwise order + TMA row
gathers); each specialisation is its own translation unit (csrc/k_inst.cu with
-DPW_DIM=d), compiled in parallel and linked with the host ABI (pw_abi.cu).

    python -m paper_2507_17094_b200.build_ext [--force]
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
OUT = PKG / "libpwb200.so"
# must match PW_DIMS / PW_DIMS_U8 / PW_DIMS_IP in csrc/pw_abi.cu (0 = generic d)
DIMS = (0, 16, 32, 64, 96, 100, 128, 200, 256, 384, 512, 768, 960, 1024)
DIMS_U8 = (0, 96, 128)
DIMS_IP = (0, 96, 128, 200)
DEPS = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "pw_b200.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed: " + " ".join(map(str, cmd)))
    return r.stderr


def build(force: bool = False, verbose: bool = False, jobs: int | None = None,
          timers: bool = False) -> Path:
    """timers=True builds libpwb200_timers.so (K1 with per-phase clock64
    counters, tools/phase_timers.py); the product library never has them."""
    out = PKG / "libpwb200_timers.so" if timers else OUT
    bdir = PKG / "_build_timers" if timers else BUILD
    if os.environ.get("PW_LIB_OUT"):  # A/B variant builds (tools/ab.py --libs)
        out = Path(os.environ["PW_LIB_OUT"]).resolve()
        bdir = out.parent / ("_build_" + out.stem)
    if not force and (out.exists() and all(p.stat().st_mtime <= out.stat().st_mtime for p in DEPS)):
        return out
    bdir.mkdir(exist_ok=True)
    nv = nvcc()
    extra = ["-DPW_PHASE_TIMERS"] if timers else []
    if os.environ.get("PW_MAX_THREADS"):  # A/B builds with more resident warps per SM
        extra.append(f"-DPW_MAX_THREADS={int(os.environ['PW_MAX_THREADS'])}")
    extra += os.environ.get("PW_EXTRA_NVCC", "").split()  # A/B build variants (-DPW_...)
    jobs_list = [([nv, *CFLAGS, *extra, "-c", str(CSRC / "pw_abi.cu"), "-o", str(bdir / "pw_abi.o")],
                  bdir / "pw_abi.o"),
                 ([nv, *CFLAGS, *extra, "-c", str(CSRC / "pw_crc32c.cu"), "-o", str(bdir / "pw_crc32c.o")],
                  bdir / "pw_crc32c.o"),
                 ([nv, *CFLAGS, *extra, "-c", str(CSRC / "knn_screen.cu"), "-o", str(bdir / "knn_screen.o")],
                  bdir / "knn_screen.o"),
                 ([nv, *CFLAGS, *extra, "-c", str(CSRC / "gather_probe.cu"), "-o", str(bdir / "gather_probe.o")],
                  bdir / "gather_probe.o")]
    # every specialised d also gets its FAST instance (-DPW_FAST, cold paths
    # compiled out; the host picks it per launch)
    for kind, dims, flag in (("", DIMS, []), ("u8_", DIMS_U8, ["-DPW_U8"]), ("ip_", DIMS_IP, ["-DPW_IP"])):
        for d in dims:
            for var, vflags in ((("", []), ("f_", ["-DPW_FAST"]), ("fw_", ["-DPW_FAST", "-DPW_WIDE"]))
                                 if d else (("", []),)):
                obj = bdir / f"k_{kind}{var}{d}.o"
                jobs_list.append(([nv, *CFLAGS, *extra, f"-DPW_DIM={d}", *flag, *vflags,
                                   "-c", str(CSRC / "k_inst.cu"), "-o", str(obj)], obj))
    workers = jobs or max(1, min(len(jobs_list), os.cpu_count() or 1))
    with ThreadPoolExecutor(workers) as pool:
        logs = list(pool.map(lambda j: _run(j[0]), jobs_list))
    objs = [str(o) for _, o in jobs_list]
    _run([nv, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(out) + ".tmp", *objs])
    os.replace(str(out) + ".tmp", out)
    if not timers and out == OUT:
        (PKG / "build_ptxas.log").write_text("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, timers="--timers" in sys.argv))
