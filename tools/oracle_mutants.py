#!/usr/bin/env python3
"""Mutation check of the oracle pins.

Each mutation is a one-line edit of oracle/sf_oracle.c (a dropped term, a flipped sign, branch or
index, a transposed operand).  For each: apply it, rebuild the oracle, run the CPU pin suites
(tests/test_oracle_*.py), restore.  A mutation must make at least one pin fail ("caught").

    python tools/oracle_mutants.py            # all mutations
    python tools/oracle_mutants.py clamp tie  # those whose label contains any of the words
"""
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "sf_oracle.c")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_branches.py", "tests/test_oracle_eval.py",
        "tests/test_oracle_pyramid.py", "tests/test_oracle_map.py", "tests/test_oracle_imu.py"]

# (label, old text, new text, occurrence): occurrence = index of the match to edit (None = all)
MUTATIONS = [
    # ---- H = 1 filter
    ("dominant neighbour swapped (PRINTED)", "uh = (FABS(up) - FABS(um) > R(0)) ? um : up;", "uh = (FABS(up) - FABS(um) > R(0)) ? up : um;", 0),
    ("dominant LARGEST picks smaller", "uh = (FABS(um) > FABS(up)) ? um : up; /*", "uh = (FABS(um) < FABS(up)) ? um : up; /*", 0),
    ("LARGEST tie -> u_{j-1}", "uh = (FABS(um) > FABS(up)) ? um : up; /*", "uh = (FABS(um) >= FABS(up)) ? um : up; /*", 0),
    ("upwind side swapped", "const real D = (uh > R(0)) ? (f[c] - fm[c]) : (fp[c] - f[c]);", "const real D = (uh > R(0)) ? (fp[c] - f[c]) : (f[c] - fm[c]);", 0),
    ("clamp removed", "uh = FMIN(FMAX(uh, -U), U);", "(void)0;", 0),
    ("clamp widened to 2U", "uh = FMIN(FMAX(uh, -U), U);", "uh = FMIN(FMAX(uh, -R(2) * U), R(2) * U);", 0),
    ("FLAG_CLAMPED dropped", "if (FABS(uh) > U) flags |= OR_FLAG_CLAMPED;", "(void)0;", 0),
    ("FLAG_CFL dropped", "} else if (dt * FABS(uh) > R(1)) {\n                flags |= OR_FLAG_CFL;", "} else if (0) {\n                flags |= OR_FLAG_CFL;", 0),
    ("source term dropped", "out[c] = FMA(-dt, FMA(uh, D, f[c] * q), f[c]);", "out[c] = FMA(-dt, uh * D, f[c]);", 0),
    ("source weight sigma = 1", "const real q = sigma * sw;", "const real q = sw;", 0),
    ("e1/e2 transposed", "u[p] = dot3(geo + 10 * p + 3 + 3 * axis, w + 3 * p);", "u[p] = dot3(geo + 10 * p + 6 - 3 * axis, w + 3 * p);", 0),
    ("row-neighbour index", "pm = (long)clampi(i - 1, 0, H - 1) * W + j;\n                pp = (long)clampi(i + 1, 0, H - 1) * W + j;\n            }\n            const real um = u[pm], up = u[pp];\n            real uh;\n            if (P->dominant_rule == OR_DOM_PRINTED)\n                uh = (FABS(up) - FABS(um) > R(0)) ? um : up; /* as",
     "pm = (long)clampi(i - 1, 0, H - 1) * W + j;\n                pp = (long)clampi(i + 2, 0, H - 1) * W + j;\n            }\n            const real um = u[pm], up = u[pp];\n            real uh;\n            if (P->dominant_rule == OR_DOM_PRINTED)\n                uh = (FABS(up) - FABS(um) > R(0)) ? um : up; /* as", 0),
    ("gradient sign flipped", "for (int a = 0; a < 3; ++a) ghat[3 * p + a] = d2 * FMA(e2[a], beta2[p], e1[a] * beta1[p]);", "for (int a = 0; a < 3; ++a) ghat[3 * p + a] = -d2 * FMA(e2[a], beta2[p], e1[a] * beta1[p]);", 0),
    ("rho side larger", "if (hp && hm) return (FABS(dp) <= FABS(dm)) ? dp : dm;", "if (hp && hm) return (FABS(dp) >= FABS(dm)) ? dp : dm;", 0),
    ("rho tie -> backward", "if (hp && hm) return (FABS(dp) <= FABS(dm)) ? dp : dm;", "if (hp && hm) return (FABS(dp) < FABS(dm)) ? dp : dm;", 0),
    ("only-forward fallback zeroed", "if (hp) return dp;", "if (hp) return R(0);", 0),
    ("only-backward fallback zeroed", "if (hm) return dm;", "if (hm) return R(0);", 0),
    ("lambda = 0 valid", "(isfinite(x) && x > R(0));", "(isfinite(x) && x >= R(0));", 0),
    ("validity ignored", "if (!v[p]) return R(0);\n    const int hp = v[pp], hm = v[pm];", "const int hp = 1, hm = 1;", 0),
    ("cY sign", "const real cY = d2 * (yh1[p] - yhat[p]);", "const real cY = d2 * (yhat[p] - yh1[p]);", 0),
    ("normal term of m dropped", "m[a] = FMA(d2r, s[a], drho[3 * p + a]);", "m[a] = drho[3 * p + a];", 0),
    ("bottom normal term of m dropped", "m[a] = FMA(d2r, s[a], drho[3 * p + a]);", "m[a] = drho[3 * p + a];", 1),
    ("E_t as printed (+)", "b[a] = FMA(-g2m[a], cr, FMA(-g1g[a], cY, g3 * wp[a]));", "b[a] = FMA(-g2m[a], cr, FMA(-g1g[a], cY, -g3 * wp[a]));", 0),
    ("box / 24", "acc / R(25);", "acc / R(24);", 0),
    ("fusion weights swapped", "const real kap = R(P->gamma[3]) / (R(P->gamma[3]) + R(P->gamma[4]));\n        real* wls",
     "const real kap = R(P->gamma[4]) / (R(P->gamma[3]) + R(P->gamma[4]));\n        real* wls", 0),
    ("d2 = ds", "o[9] = ds * ds;", "o[9] = ds;", 0),
    # ---- NEXT rows
    ("tangent flow e2 first", "tangent[2 * p] = dot3(g + 3, t);", "tangent[2 * p] = dot3(g + 6, t);", 0),
    ("normal / ds^2", "if (normal) normal[p] = sw / ds;", "if (normal) normal[p] = sw / (ds * ds);", 0),
    ("projection sign", "for (int a = 0; a < 3; ++a) t[a] = FMA(-g[a], sw, wp[a]);", "for (int a = 0; a < 3; ++a) t[a] = FMA(g[a], sw, wp[a]);", 0),
    ("RMSE without / ds", "d[k] = (wgt[3 * p + k] - w[3 * p + k]) / ds;", "d[k] = (wgt[3 * p + k] - w[3 * p + k]);", 0),
    ("AAE without the homogeneous 1", "double c = (1.0 + ddot3(a, b)) / (sqrt(1.0 + ddot3(a, a)) * sqrt(1.0 + ddot3(b, b)));",
     "double c = (ddot3(a, b)) / (sqrt(ddot3(a, a)) * sqrt(ddot3(b, b)));", 0),
    ("2x2 mean weight", "if (Y2) Y2[o] = ((Y[a] + Y[a + 1]) + (Y[b] + Y[b + 1])) * 0.25f;", "if (Y2) Y2[o] = ((Y[a] + Y[a + 1]) + (Y[b] + Y[b + 1])) * 0.5f;", 0),
    ("up-sampling row weights swapped", "const real wr0 = (i & 1) ? R(0.75) : R(0.25), wr1 = (i & 1) ? R(0.25) : R(0.75);",
     "const real wr0 = (i & 1) ? R(0.25) : R(0.75), wr1 = (i & 1) ? R(0.75) : R(0.25);", 0),
    ("Yhat dilated at the bottom level", "Fo[8 * p + c] = (c < 7) ? FMA(-dt, FMA(uh, D, f * q), f) : FMA(-dt, uh * D, f);",
     "Fo[8 * p + c] = FMA(-dt, FMA(uh, D, f * q), f);", 0),
    ("bottom clamp removed", "uh = FMIN(FMAX(uh, -U), U);", "(void)0;", 1),
    ("increment update: rho reference rho^k", "const real cr = d2 * (rh[p] - F[8 * p + 6]);", "const real cr = d2 * (rh[p] - S->rho2[0]);", 0),
    ("bottom prior = w instead of dw", "ls_solve(ghat + 3 * p, m, cY, cr, F + 8 * p + 3,", "ls_solve(ghat + 3 * p, m, cY, cr, F + 8 * p + 0,", 0),
    ("bottom cY sign", "const real cY = d2 * (yh1[p] - F[8 * p + 7]);", "const real cY = d2 * (F[8 * p + 7] - yh1[p]);", 0),
    ("bottom fusion dropped", "F[8 * p + 6] = FMA(kappa, rh[p] - F[8 * p + 6], F[8 * p + 6]);", "(void)0;", 0),
    ("reconstruction without dw", "F[8 * p + a] = up[3 * p + a] + F[8 * p + 3 + a];", "F[8 * p + a] = up[3 * p + a];", 0),
    ("mapping f_y for u", "u = fmaf(fx, t[0] / t[2], cx);", "u = fmaf(fy, t[0] / t[2], cx);", 0),
    ("z-depth not converted to range", "D[p] = fmaf(a, r1 - r0, r0) / t[2];", "D[p] = fmaf(a, r1 - r0, r0);", 0),
    ("bilinear weights swapped", "const float r0 = fmaf(b, Ycam[q01] - Ycam[q00], Ycam[q00]);", "const float r0 = fmaf(a, Ycam[q01] - Ycam[q00], Ycam[q00]);", 0),
    ("Coriolis factor 1", "const real f = FMA(rho[p], ac[a], -FMA(R(2), c3[a], c2[a]));", "const real f = FMA(rho[p], ac[a], -FMA(R(1), c3[a], c2[a]));", 0),
    ("acceleration sign", "const real f = FMA(rho[p], ac[a], -FMA(R(2), c3[a], c2[a]));", "const real f = FMA(rho[p], -ac[a], -FMA(R(2), c3[a], c2[a]));", 0),
    ("centripetal dropped", "const real f = FMA(rho[p], ac[a], -FMA(R(2), c3[a], c2[a]));", "const real f = FMA(rho[p], ac[a], -(R(2) * c3[a]));", 0),
]


def apply(src, old, new, occ):
    idx = [m.start() for m in re.finditer(re.escape(old), src)]
    if not idx:
        return None
    if occ is None:
        return src.replace(old, new)
    if occ >= len(idx):
        return None
    i = idx[occ]
    return src[:i] + new + src[i + len(old):]


def main():
    words = sys.argv[1:]
    orig = open(SRC).read()
    backup = SRC + ".orig"
    shutil.copy(SRC, backup)
    results = []
    try:
        for label, old, new, occ in MUTATIONS:
            if words and not any(w.lower() in label.lower() for w in words):
                continue
            mutated = apply(orig, old, new, occ)
            if mutated is None:
                results.append((label, "DID NOT APPLY"))
                print(f"{label}: DID NOT APPLY", flush=True)
                continue
            open(SRC, "w").write(mutated)
            subprocess.run([sys.executable, os.path.join(ROOT, "oracle", "build.py"), "--force"], check=True,
                           capture_output=True, cwd=ROOT)
            r = subprocess.run([sys.executable, "-m", "pytest", *PINS, "-q", "-p", "no:cacheprovider"], cwd=ROOT,
                               capture_output=True, text=True, timeout=1800)
            tail = (r.stdout.strip().splitlines() or ["?"])[-1]
            m = re.search(r"(\d+) failed", tail)
            verdict = f"caught ({m.group(1)} pins fail)" if m else ("SURVIVED" if r.returncode == 0 else f"error: {tail}")
            results.append((label, verdict))
            print(f"{label}: {verdict}", flush=True)
    finally:
        open(SRC, "w").write(orig)
        os.remove(backup)
        subprocess.run([sys.executable, os.path.join(ROOT, "oracle", "build.py"), "--force"], check=True,
                       capture_output=True, cwd=ROOT)
    bad = [l for l, v in results if not v.startswith("caught")]
    print(f"\n{len(results) - len(bad)}/{len(results)} mutations caught" + (f"; NOT caught: {bad}" if bad else ""))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
