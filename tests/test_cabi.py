"""The C-ABI library loads on a CPU-only host and exports every entry point that
include/driftcast_gpu.h declares (no compute calls: there is no GPU here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "driftcast_gpu.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(dc_[A-Za-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    from paper_1910_01031_b200 import _lib
    L = _lib.load()
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == names, set(_lib.EXPORTS) ^ set(names)


def test_version_string_without_gpu():
    from paper_1910_01031_b200 import _lib
    L = _lib.load()
    assert b"sm_100a" in L.dc_version()


def test_library_is_sm100a_native():
    """The fatbin carries sm_100a SASS (cuobjdump), not PTX-only or another arch."""
    import shutil
    import subprocess
    so = os.path.join(ROOT, "paper_1910_01031_b200", "libdriftcast_gpu.so")
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_validation_without_gpu():
    """Parameter checks mirror the reference constructors and run before any CUDA call."""
    from paper_1910_01031_b200 import Config, _lib
    L = _lib.load()
    bad = [Config(nx=4), Config(c_omega=4), Config(c_omega=7), Config(courant=1.5),
           Config(f=0.0), Config(h_eq=-1.0)]
    for cfg in bad:
        c = cfg.to_c()
        h = C.c_void_p()
        rc = L.dc_create(C.byref(c), 2, 0, 0, None, C.byref(h))
        assert rc == 1, cfg  # DC_EINVAL


def test_precompute_on_host_matches_oracle(oracle):
    """dc_precompute_S / dc_precompute_local_svd run on the host (no GPU needed) and
    agree with the CPU restatement bit-for-bit (block) / to reconstruction (U Sigma^1/2)."""
    import numpy as np
    from checkers import make_params
    from paper_1910_01031_b200 import Config, precompute_S, precompute_local_svd
    cfg = Config()
    p = make_params()
    h, S = precompute_S(cfg)
    ho, So = oracle.precompute_S(p, 0, 0)
    assert np.array_equal(h, ho) and np.array_equal(S, So)
    blk, usig = precompute_local_svd(cfg, S)
    assert np.array_equal(blk, oracle.local_block(p, S))
    assert np.abs(usig @ usig.T - blk).max() < 1e-12
