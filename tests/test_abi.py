"""CPU-only checks of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/glmb.h declares, and its host-side validation answers without a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "glmb.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2512_06230_b200.build import build
    path = build()
    return C.CDLL(path), path


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(glmb_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_four_calls():
    names = declared_functions()
    for n in ("glmb_predict", "glmb_birth", "glmb_compat", "glmb_reweight"):
        assert n in names


def test_exports_every_declared_symbol(lib):
    L, path = lib
    names = declared_functions()
    for n in names:
        assert hasattr(L, n), f"{n} missing from {path}"
    nm = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (glmb_\w+)", nm))
    assert set(names) <= exported
    from paper_2512_06230_b200 import _lib
    assert set(_lib.EXPORTED) == set(names)


def test_sm100a_cubin_inside(lib):
    _, path = lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", path], capture_output=True,
                          text=True).stdout
    for mnem in ("MUFU.EX2", "FFMA2", "FADD2", "UBLKCP", "SYNCS"):
        assert mnem in sass, f"{mnem} not found in the SASS"


def test_status_strings_and_version(lib):
    L, _ = lib
    L.glmb_status_string.restype = C.c_char_p
    for s in (0, -1, -2, -3, -4):
        assert L.glmb_status_string(s).decode().startswith("GLMB_")
    assert L.glmb_version() == 10000


def test_validation_without_gpu(lib):
    """Argument checks run on the host before any CUDA call."""
    L, _ = lib
    from paper_2512_06230_b200._lib import glmb_particles
    fake = 0x1000  # never dereferenced: validation fails first
    p = glmb_particles(fake, fake, fake, fake, fake, fake, 2, 8, 8)
    f32 = C.c_float
    L.glmb_compat.argtypes = [C.POINTER(glmb_particles), C.c_void_p, C.c_int32] + [f32] * 6 + [
        C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]
    # R not SPD
    assert L.glmb_compat(C.byref(p), fake, 3, 1.0, 2.0, 1.0, 0.9, 1e-3, 1e-6, None, fake, 3, fake, 1, None) == -1
    # P_D out of range, kappa < 0, gamma below 1e-30
    assert L.glmb_compat(C.byref(p), fake, 3, 1.0, 0.0, 1.0, 1.5, 1e-3, 1e-6, None, fake, 3, fake, 1, None) == -1
    assert L.glmb_compat(C.byref(p), fake, 3, 1.0, 0.0, 1.0, 0.9, -1.0, 1e-6, None, fake, 3, fake, 1, None) == -1
    assert L.glmb_compat(C.byref(p), fake, 3, 1.0, 0.0, 1.0, 0.9, 1e-3, 1e-31, None, fake, 3, fake, 1, None) == -1
    # ldc < M, ldg too small
    assert L.glmb_compat(C.byref(p), fake, 40, 1.0, 0.0, 1.0, 0.9, 1e-3, 1e-6, None, fake, 39, fake, 2, None) == -1
    assert L.glmb_compat(C.byref(p), fake, 40, 1.0, 0.0, 1.0, 0.9, 1e-3, 1e-6, None, fake, 40, fake, 1, None) == -1
    # misaligned array / P not a multiple of 4
    bad = glmb_particles(fake + 4, fake, fake, fake, fake, fake, 2, 8, 8)
    assert L.glmb_compat(C.byref(bad), fake, 3, 1.0, 0.0, 1.0, 0.9, 1e-3, 1e-6, None, fake, 3, fake, 1, None) == -2
    odd = glmb_particles(fake, fake, fake, fake, fake, fake, 2, 6, 8)
    assert L.glmb_compat(C.byref(odd), fake, 3, 1.0, 0.0, 1.0, 0.9, 1e-3, 1e-6, None, fake, 3, fake, 1, None) == -2
    # predict: dt <= 0
    L.glmb_predict.argtypes = [C.POINTER(glmb_particles)] * 2 + [C.c_void_p, f32, f32, f32, C.c_uint64,
                                                                 C.c_uint32, C.c_void_p]
    assert L.glmb_predict(C.byref(p), C.byref(p), fake, 0.0, 1.0, 0.1, 0, 0, None) == -1
    assert L.glmb_predict(C.byref(p), C.byref(p), None, 0.1, 1.0, 0.1, 0, 0, None) == -1
    # empty inputs are successful no-ops (no device touched)
    empty = glmb_particles(None, None, None, None, None, None, 0, 8, 8)
    assert L.glmb_predict(C.byref(empty), C.byref(empty), None, 0.1, 1.0, 0.1, 0, 0, None) == 0
    assert L.glmb_compat(C.byref(p), None, 0, 1.0, 0.0, 1.0, 0.9, 1e-3, 1e-6, None, None, 0, None, 0, None) == 0


def test_validation_hypothesis_calls_without_gpu():
    """The f1-f4 entry points reject bad arguments on the host (status -1 / -2) and treat
    empty work as a successful no-op, before any CUDA call."""
    from paper_2512_06230_b200 import _lib
    L = _lib.load()
    fake = 0x1000
    # death_prob: p_d out of range, kappa < 0, ldc < M
    assert L.glmb_death_prob(3, 40, fake, 40, fake, 2, 1.5, 1e-3, fake, fake, None) == -1
    assert L.glmb_death_prob(3, 40, fake, 40, fake, 2, 0.9, -1.0, fake, fake, None) == -1
    assert L.glmb_death_prob(3, 40, fake, 39, fake, 2, 0.9, 1e-3, fake, fake, None) == -1
    assert L.glmb_death_prob(0, 40, None, 0, None, 0, 0.9, 1e-3, None, None, None) == 0
    # compat_rows: NULL row_ptr, NULL outputs with cap > 0
    assert L.glmb_compat_rows(3, 40, fake, 40, fake, 2, None, fake, fake, fake, 8, None) == -1
    assert L.glmb_compat_rows(3, 40, fake, 40, fake, 2, fake, None, fake, fake, 8, None) == -1
    # assoc_sample: H_up >= 2^24, ldt too small, misaligned theta / ldm % 4, count prior without a table
    args = lambda **kw: dict(dict(H_old=2, n_par=None, H_up=8, T=40, M=10, pm=fake, ldt=2, plw=fake, d=fake,
                                  ps=fake, pd=0.9, kappa=1e-3, rp=fake, col=fake, val=fake, lv=fake, clp=None,
                                  ncount=0, seed=0, step=0, alive=fake, theta=fake, ldm=12, logw=fake,
                                  hash=None, s=None), **kw)
    call = lambda a: L.glmb_assoc_sample(*a.values())
    assert call(args(H_up=1 << 24)) == -1
    assert call(args(ldt=1)) == -1
    assert call(args(ldm=10)) == -2
    assert call(args(theta=fake + 4)) == -2
    assert call(args(ncount=3)) == -1
    assert call(args(H_old=0)) == 0
    # dedup / prune
    assert L.glmb_dedup(2, None, 8, 10, fake, 0, fake, 12, fake, fake, None) == -1      # ldt < 1
    assert L.glmb_prune(10, fake, fake, -1.0, 5, fake, fake, fake, fake, None) == -1    # tau < 0
    assert L.glmb_prune(10, fake, fake, 0.0, 16385, fake, fake, fake, fake, None) == -1  # h_max > limit
    # pairs / particle loop
    assert L.glmb_assoc_pairs(2, None, fake, fake, 2, fake, 12, 40, 10, fake, fake, fake, fake, fake,
                              fake, 1, None) == -1                                     # short workspace
    assert L.glmb_assoc_pairs_workspace_size(-1, 4, 4) == 0
    p = _lib.glmb_particles(fake, fake, fake, fake, fake, fake, 2, 8, 8)
    big = _lib.glmb_particles(fake, fake, fake, fake, fake, fake, 2, 16388, 16388)
    assert L.glmb_reweight_pairs(C.byref(big), fake, 3, 1.0, 0.0, 1.0, 4, None, fake, fake, fake, fake, 16388,
                                 fake, fake, fake, None) == -1                         # P > GLMB_PAIRS_PMAX
    assert L.glmb_reweight_pairs(C.byref(p), fake, 3, 1.0, 0.0, 1.0, 4, None, fake, fake, fake, fake + 4, 8,
                                 fake, fake, fake, None) == -2                         # misaligned w_out
    assert L.glmb_reweight_pairs(C.byref(p), fake, 3, 1.0, 0.0, 1.0, 0, None, None, None, None, None, 8,
                                 None, None, None, None) == 0                          # K = 0
    assert L.glmb_resample(C.byref(p), 2, None, fake, fake, 6, C.byref(p), 0, 0, None, None) == -2   # ldw % 4
    assert L.glmb_resample(C.byref(p), 3, None, fake, fake, 8, C.byref(p), 0, 0, None, None) == -1   # out too small
    # tracker loop
    assert L.glmb_next_parents(4, fake, fake, fake, 10, 64, 1, 0, fake, 1, fake, fake, None, None) == -1  # K_cap > 32 ldt
    assert L.glmb_next_parents(4, fake, fake, fake, 10, 32, 1, 0, fake, 1, fake, fake, fake, None) == -1  # K_cap + B > 32 ldt (device col0)
    assert L.glmb_map_estimate(None, fake, 3, C.byref(p), fake, None) == -1
