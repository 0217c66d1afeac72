"""Build the C oracle (TEST INFRASTRUCTURE ONLY) into oracle/liboracle_{f32,f64}.so.

Plain gcc, -O2 -ffp-contract=off (no implicit contraction; the oracle's fused
multiply-adds are explicit fma() calls), no -march tuning, single-threaded.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sf_oracle.c")
FLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall", "-Wextra", "-Wno-maybe-uninitialized"]


def lib_path(prec: str) -> str:
    return os.path.join(HERE, f"liboracle_{prec}.so")


def build(force: bool = False) -> None:
    for prec, defs in (("f32", ["-DOR_F32"]), ("f64", [])):
        out = lib_path(prec)
        if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(SRC):
            continue
        cmd = ["gcc", *FLAGS, *defs, SRC, "-o", out, "-lm"]
        subprocess.run(cmd, check=True)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print("built", lib_path("f32"), lib_path("f64"))
