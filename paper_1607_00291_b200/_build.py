"""Build libtc_b200.so in-tree with nvcc for sm_100a (called by __graft_entry__.build()).

Each translation unit is compiled to an object in parallel (the kernel instantiations are split
over ws_*.cu), then linked into one shared library."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# TC_LIB_OUT / TC_NVCC_EXTRA: build a variant library elsewhere with extra nvcc flags (kernel
# A/B experiments, e.g. -DTC_STAGES_F32=4); load it with TC_B200_LIB=<path>.
LIB = os.environ.get("TC_LIB_OUT") or os.path.join(HERE, "libtc_b200.so")
OBJ = os.path.join(HERE, "build_obj") if not os.environ.get("TC_LIB_OUT") else LIB + ".obj"
EXTRA = os.environ.get("TC_NVCC_EXTRA", "").split()
SOURCES = ["plan.cpp", "tc_api.cpp", "contract_kernels.cu", "skinny.cu", "tiny.cu", "rankk.cu", "umma_f32.cu", "umma_f32_n256.cu", "umma_f32_pair.cu",
           "ws_f64_a0.cu", "ws_f64_a1.cu", "ws_f64_a2.cu",
           "ws_f32_ffma_a0.cu", "ws_f32_ffma_a1.cu", "ws_f32_ffma_a2.cu", "ws_f32_ffma_a3.cu",
           "ws_f32_dmma.cu"]
HEADERS = ["plan.hpp", "kernels.hpp", "dev_common.cuh", "contract_ws.cuh", "sched.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def _deps_mtime() -> float:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "tc.h")]
    return max(os.path.getmtime(d) for d in deps if os.path.exists(d))


def _stale() -> bool:
    return not os.path.exists(LIB) or os.path.getmtime(LIB) < _deps_mtime()


def _compile(nvcc: str, src: str):
    obj = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
    cmd = [nvcc, *NVCC_FLAGS, *EXTRA, "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c",
           os.path.join(CSRC, src), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, cmd, res


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    os.makedirs(OBJ, exist_ok=True)
    log = []
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(nvcc, s), SOURCES))
    failed = False
    for src, obj, cmd, res in results:
        log.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            failed = True
            sys.stderr.write(res.stderr[-6000:])
    tmp = LIB + f".tmp{os.getpid()}"
    if not failed:
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
               *[r[1] for r in results], "-o", tmp, "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        failed = res.returncode != 0
        if failed:
            sys.stderr.write(res.stderr[-6000:])
    with open(os.path.join(HERE, "build.log") if LIB.startswith(HERE) else LIB + ".log", "w") as f:
        f.write("\n".join(log))
    if failed:
        raise RuntimeError("nvcc build of libtc_b200.so failed (see paper_1607_00291_b200/build.log)")
    if verbose:
        sys.stderr.write("\n".join(log))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
