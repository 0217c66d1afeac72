"""The C-ABI library loads and exports every symbol include/sf.h declares; the ctypes
config layout matches the C struct; host-side validation works without a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sf.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sf_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("sf_create", "sf_predict", "sf_update", "sf_step", "sf_get_fields"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2406_18031_b200 as sf

    lib = C.CDLL(sf.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(sf.EXPORTS) == set(_declared())
    out = subprocess.run(["nm", "-D", "--defined-only", sf.LIB_PATH], capture_output=True, text=True).stdout
    for n in _declared():
        assert re.search(rf"\bT {n}\b", out), n


def test_config_layout_matches_header(tmp_path):
    import paper_2406_18031_b200 as sf

    prog = tmp_path / "layout.c"
    fields = [f[0] for f in sf.sf_config._fields_]
    body = "".join(f'printf("{f} %zu\\n", offsetof(sf_config, {f}));' for f in fields)
    prog.write_text(f'#include <stdio.h>\n#include <stddef.h>\n#include "sf.h"\nint main(void){{{body}'
                    f'printf("size %zu\\n", sizeof(sf_config));return 0;}}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.dirname(HEADER), str(prog), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")
               if line)
    for f in fields:
        assert int(got[f]) == getattr(sf.sf_config, f).offset, f
    assert int(got["size"]) == C.sizeof(sf.sf_config)


def test_validation_without_gpu():
    """Invalid configurations are rejected synchronously, before any CUDA call."""
    import numpy as np

    import paper_2406_18031_b200 as sf

    g = np.zeros((8, 8, 10), np.float32)
    cases = [("height", 1, sf.SF_E_CONFIG), ("batch", 0, sf.SF_E_CONFIG), ("max_flow_px", 0.0, sf.SF_E_CONFIG),
             ("smooth_iters", -1, sf.SF_E_CONFIG), ("dominant_rule", 7, sf.SF_E_CONFIG),
             ("levels", 3, sf.SF_E_UNSUPPORTED), ("levels", 0, sf.SF_E_UNSUPPORTED), ("abi_version", 99, sf.SF_E_CONFIG)]
    for field, val, want in cases:
        cfg = sf.sf_config_default(8, 8)
        setattr(cfg, field, val)
        with pytest.raises(sf.SFError) as e:
            sf.sf_create(cfg, g.ctypes.data)
        assert e.value.status == want, field
    # pyramid: even sizes >= 4, smooth_iters_top in [0, 64], no banded mode
    for (h, w, field, val, want) in [(10, 9, None, None, sf.SF_E_CONFIG), (8, 8, "smooth_iters_top", -1, sf.SF_E_CONFIG),
                                     (2, 8, None, None, sf.SF_E_CONFIG)]:
        cfg = sf.sf_config_default(h, w)
        cfg.levels = 2
        if field:
            setattr(cfg, field, val)
        with pytest.raises(sf.SFError) as e:
            sf.sf_create(cfg, g.ctypes.data)
        assert e.value.status == want, (h, w, field)
    cfg = sf.sf_config_default(8, 8)
    cfg.gamma[2] = 0.0  # gamma3 must be > 0 (A SPD)
    with pytest.raises(sf.SFError) as e:
        sf.sf_create(cfg, g.ctypes.data)
    assert e.value.status == sf.SF_E_CONFIG
    with pytest.raises(sf.SFError) as e:
        sf.sf_create(sf.sf_config_default(8, 8), 0)
    assert e.value.status == sf.SF_E_DATA
    for call in (lambda: sf.sf_predict(0), lambda: sf.sf_step(0, 1, 1), lambda: sf.sf_get_fields(0, 0, 0, 0, 0)):
        with pytest.raises(sf.SFError) as e:
            call()
        assert e.value.status == sf.SF_E_DATA
    assert "configuration" in sf.sf_error_string(sf.SF_E_CONFIG)


def test_product_package_does_not_touch_the_oracle():
    """The CUDA path never imports oracle/ (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_2406_18031_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b|liboracle|sf_oracle|#include.*oracle", txt,
                                     re.M), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2406_18031_b200|libsf|#include.*sf\.h", txt, re.M), f
