"""In-tree build of the native libraries (no torch JIT cache, no pip install).

  paper_2310_09259_b200/lib/libquik_b200.so   product: sm_100a kernels + C ABI
  oracle/build/libquik_oracle.so              test oracle (plain C restatement)
  oracle/_ref/libquik_ref.so                  the reference's own sources + a C shim
                                              (only when /root/reference is present)

The .so files are git-ignored but travel to the GPU box with the repo snapshot.
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
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libquik_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                     "-I" + str(ROOT / "include")]
SOURCES = ["gemm.cu", "stream4.cu", "wo.cu", "gptq.cu", "quantize.cu", "weights.cu", "capi.cu", "bundle.cpp"]


def _run(cmd: list[str], cwd: Path | None = None) -> None:
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} ... {cmd[-1]}")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_product(force: bool = False) -> Path:
    LIBDIR.mkdir(exist_ok=True)
    objdir = ROOT / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h"))
    jobs = []
    objs = []
    for s in SOURCES:
        src = CSRC / s
        obj = objdir / (s + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()
    if force or jobs or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-cudart", "shared",
              "-Xlinker", "-soname=libquik_b200.so"])
    return LIB


def build_oracle(force: bool = False) -> Path:
    odir = ROOT / "oracle"
    out = odir / "build" / "libquik_oracle.so"
    out.parent.mkdir(exist_ok=True)
    src = odir / "quik_oracle.c"
    if force or _stale(out, [src, odir / "quik_oracle.h"]):
        _run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
              "-Wall", str(src), "-o", str(out), "-lm"])
    return out


REF_SRC = Path("/root/reference/proj")


def build_reference(force: bool = False) -> Path | None:
    """Compiles the reference's own arithmetic (packed/calibration/quantizer/runtime.cpp)
    with its Release flags (CMakeLists.txt:11-13) plus oracle/ref_shim.cpp into
    oracle/_ref/libquik_ref.so. Skipped when /root/reference is absent (GPU box)."""
    odir = ROOT / "oracle"
    out = odir / "_ref" / "libquik_ref.so"
    if not REF_SRC.exists():
        return out if out.exists() else None
    out.parent.mkdir(exist_ok=True)
    srcs = [REF_SRC / "src" / f for f in ("packed.cpp", "calibration.cpp", "quantizer.cpp", "runtime.cpp",
                                            "container.cpp", "layer_io.cpp")]
    shim = odir / "ref_shim.cpp"
    # the container / layer-bundle sources include <json.hpp> (nlohmann 3.x, vendored in
    # the reference's absent vendor dir; the same header ships with cudnn_frontend here)
    json_dir = Path(sys.prefix) / "lib" / f"python{sys.version_info.major}.{sys.version_info.minor}" / \
        "site-packages" / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
    if force or _stale(out, srcs + [shim]):
        _run(["g++", "-std=c++20", "-O3", "-DNDEBUG", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
              "-I" + str(REF_SRC / "include"), "-I" + str(json_dir), *map(str, srcs), str(shim), "-o", str(out)])
    return out


def build_tests(force: bool = False) -> Path:
    """C++ parity driver for the drop-in facade (include/quik_b200.hpp); test
    infrastructure: links the product library and the oracle (as the checker)."""
    src = ROOT / "tests" / "cpp" / "facade_test.cpp"
    out = ROOT / "build" / "tests" / "facade_test"
    out.parent.mkdir(parents=True, exist_ok=True)
    deps = [src, ROOT / "include" / "quik_b200.hpp", ROOT / "include" / "quik_b200.h", LIB,
            ROOT / "oracle" / "build" / "libquik_oracle.so"]
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O2", "-Wall", "-I" + str(ROOT / "include"), "-I/usr/local/cuda/include",
              str(src), "-o", str(out), "-L" + str(LIBDIR), "-lquik_b200",
              str(ROOT / "oracle" / "build" / "libquik_oracle.so"), "-L/usr/local/cuda/lib64", "-lcudart",
              "-Wl,-rpath," + str(LIBDIR), "-Wl,-rpath,$ORIGIN/../../paper_2310_09259_b200/lib",
              "-Wl,-rpath,$ORIGIN/../../oracle/build", "-Wl,-rpath," + str(ROOT / "oracle" / "build")])
    return out


def build_ipc_test(force: bool = False) -> Path:
    """C++ two-process test of the fused all-gather through CUDA IPC (FusedShardedLayer)."""
    src = ROOT / "tests" / "cpp" / "ipc_test.cpp"
    out = ROOT / "build" / "tests" / "ipc_test"
    out.parent.mkdir(parents=True, exist_ok=True)
    deps = [src, ROOT / "include" / "quik_b200.hpp", ROOT / "include" / "quik_b200.h", LIB]
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O2", "-Wall", "-I" + str(ROOT / "include"), "-I/usr/local/cuda/include",
              str(src), "-o", str(out), "-L" + str(LIBDIR), "-lquik_b200", "-L/usr/local/cuda/lib64", "-lcudart",
              "-Wl,-rpath," + str(LIBDIR), "-Wl,-rpath,$ORIGIN/../../paper_2310_09259_b200/lib"])
    return out


def build_all(force: bool = False) -> None:
    build_product(force)
    build_oracle(force)
    build_reference(force)
    build_tests(force)
    build_ipc_test(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built", LIB)
