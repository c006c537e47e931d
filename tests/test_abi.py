"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/lsk.h
declares, and its host logic (Lambert W_0, shard ranges, argument validation) is right.
No compute kernel is launched here."""
import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest
import scipy.special

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "lsk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lsk_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    import paper_2006_07057_b200 as L
    declared = _header_functions()
    assert len(declared) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    # the binding wraps exactly the declared API
    assert set(L.EXPORTED) == set(declared)


def test_library_is_sm100a():
    import paper_2006_07057_b200 as L
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_lambert_w0_abi_matches_scipy():
    import paper_2006_07057_b200 as L
    for z in np.logspace(-10, 7, 300):
        w = L.lsk_lambert_w0(float(z))
        assert abs(w - float(np.real(scipy.special.lambertw(z)))) <= 1e-13 * max(1, abs(w))
    assert L.lsk_lambert_w0(0.0) == 0.0
    with pytest.raises(L.LskError):
        L.lsk_lambert_w0(-1.0)


def test_feature_params_host_only_matches_oracle():
    """R given, no points: pure host computation (a1)."""
    import oracle as O
    import paper_2006_07057_b200 as L
    for eps, d, r, R in [(0.5, 2, 100, 1.24), (0.2, 16, 2048, 1.0), (1.0, 128, 512, 1.33)]:
        p = L.lsk_feature_params_init(eps, d, r, R, 7)
        o = O.gaussian_params(eps, d, r, R)
        for k in ("q", "sigma", "log_scale"):
            assert abs(p.as_dict()[k] - o[k]) <= 1e-14 * max(1.0, abs(o[k])), k


def test_shard_range_partitions():
    import paper_2006_07057_b200 as L
    for total in (0, 1, 7, 200000, 1 << 23):
        for nr in (1, 2, 3, 4, 8):
            spans = [L.lsk_shard_range(total, nr, k) for k in range(nr)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(L.LskError):
        L.lsk_shard_range(10, 2, 2)


def test_argument_validation_without_gpu():
    import paper_2006_07057_b200 as L
    with pytest.raises(L.LskError) as e:
        L.lsk_feature_params_init(-1.0, 2, 100, 1.0, 0)
    assert e.value.status == -1
    with pytest.raises(L.LskError):
        L.lsk_feature_params_init(0.5, 2, 100, 0.0, 0)   # auto R needs points
    p = L.lsk_feature_params()
    assert L._lib.lsk_draw_anchors(ctypes.byref(p), None, None) == -1
    o = L.make_opts(10)
    rep = L.lsk_report()
    # r % 4 != 0 is rejected before any device work
    st = L._lib.lsk_factored_sinkhorn(None, 10, None, 10, 6, None, None, 0.5,
                                      ctypes.byref(o), None, None, ctypes.byref(rep), None, None)
    assert st == -1
    assert "multiple of 4" in L._lib.lsk_last_error().decode()


def test_binding_fails_loudly_without_the_library(tmp_path):
    """The product path has no CPU fallback: importing the binding with no CUDA library
    raises instead of degrading (the tuning override points at a file that does not exist)."""
    import subprocess
    import sys
    env = dict(os.environ, LSK_LIB_PATH=str(tmp_path / "missing_liblsk.so"))
    res = subprocess.run([sys.executable, "-c", "import paper_2006_07057_b200"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode != 0
    assert "ImportError" in res.stderr and "no CPU fallback" in res.stderr
