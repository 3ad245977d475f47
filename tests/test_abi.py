"""CPU checks of the C-ABI library: it builds for sm_100a, loads, and exports every symbol that
include/*.h declares (no compute calls -- there is no GPU here)."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        names += re.findall(r"^DTSDF_API\s+[\w\s\*]+?\b(dtsdf_\w+)\s*\(", open(h).read(), flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2301_12796_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("dtsdf_upload_volume", "dtsdf_render", "dtsdf_render_batch", "dtsdf_create", "dtsdf_destroy",
              "dtsdf_alloc_volume", "dtsdf_commit_volume", "dtsdf_last_error"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    for n in _declared():
        assert hasattr(lib, n), n


def test_binding_covers_the_header():
    import paper_2301_12796_b200 as pkg
    assert sorted(pkg.EXPORTS) == _declared()


def test_exported_dynamic_symbols_are_only_the_abi(lib):
    from paper_2301_12796_b200 import build
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r" T (dtsdf_\w+)", out)))
    assert exported == _declared()


def test_sass_is_sm100a(lib):
    from paper_2301_12796_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_null_context_errors_without_gpu(lib):
    """Argument checks run before any CUDA call: NULL handles fail with INVALID_ARGUMENT."""
    lib.dtsdf_last_error.restype = ctypes.c_char_p
    assert lib.dtsdf_volume_stats(None, None, None, None) == -1
    assert b"NULL" in lib.dtsdf_last_error()
    assert lib.dtsdf_set_option(None, 1, 0) == -1
    assert lib.dtsdf_destroy(None) == 0


def test_should_recombine_matches_oracle_conditions():
    """dtsdf_should_recombine (host code of the C ABI, no GPU call) agrees with the oracle's
    eqs. condition_1-4 on random pose pairs around the thresholds."""
    import numpy as np

    import oracle
    from paper_2301_12796_b200.dtsdf import should_recombine
    rng = np.random.default_rng(11)
    for _ in range(400):
        frame = int(rng.integers(0, 120))
        last = int(rng.integers(0, frame + 1))
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        ang = rng.uniform(0, 0.16)
        Kx = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
        Rr = np.eye(3) + np.sin(ang) * Kx + (1 - np.cos(ang)) * Kx @ Kx
        A = np.eye(4)
        A[:3, 3] = rng.normal(size=3)
        B = np.eye(4)
        B[:3, :3] = Rr
        B[:3, 3] = A[:3, 3] + rng.normal(size=3) / np.sqrt(3) * rng.uniform(0, 0.1)
        a = should_recombine(frame, last, B, A)
        b = oracle.should_recombine(frame, last, B, A)
        tdist = np.linalg.norm(B[:3, 3] - A[:3, 3])
        if abs(tdist - 0.05) > 1e-5 and abs(ang - 0.05 * np.pi / 2) > 1e-4:  # float32 poses at the edges
            assert a == b, (frame, last, tdist, ang)
