"""Build libsf.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python paper_2406_18031_b200/build.py [--force]   (a script: the package itself refuses to import
    without libsf.so, so the build never goes through the package __init__)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["sf_api.cu", "sf_passes.cu", "sf_fused.cu", "sf_band.cu", "sf_eval.cu", "sf_pyramid.cu", "sf_map.cu", "sf_update.cu"]
LIB = os.path.join(HERE, "libsf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC,-O2", "-shared", "-Xptxas", "-v,-warn-spills",
    # IEEE float32: no fast math, no FTZ, correctly rounded division / sqrt
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-I" + os.path.join(ROOT, "include"),
    "-ldl",
]


def _deps():
    files = [os.path.join(CSRC, s) for s in SOURCES]
    files += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    files.append(os.path.join(ROOT, "include", "sf.h"))
    return files


STAMP = os.path.join(HERE, "build_flags.txt")


def build(force: bool = False, verbose: bool = False) -> str:
    """SF_BUILD_DEBUG=1 compiles the timing / phase-skip knobs of the fused kernel (SF_DEBUG_SKIP);
    the default build folds them away."""
    extra = ["-DSF_DEBUG_KNOBS"] if os.environ.get("SF_BUILD_DEBUG") == "1" else []
    extra += os.environ.get("SF_NVCC_EXTRA", "").split()  # experiments only (e.g. -DSF_EXP_...)
    cmd = [NVCC, *FLAGS, *extra, *[os.path.join(CSRC, s) for s in SOURCES], "-o", LIB]
    same = os.path.exists(STAMP) and open(STAMP).read() == " ".join(cmd)
    if (not force and same and os.path.exists(LIB) and
            os.path.getmtime(LIB) >= max(os.path.getmtime(f) for f in _deps())):
        return LIB
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libsf.so")
    if verbose:
        sys.stderr.write(r.stderr)
    with open(os.path.join(HERE, "build_ptxas.log"), "w") as fh:
        fh.write(r.stderr)
    with open(STAMP, "w") as fh:
        fh.write(" ".join(cmd))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
