"""Comparison rules of the GPU-vs-oracle parity tests (BASELINE.json north_star;
DESIGN.md "Parity contract").  Test infrastructure only."""
import math

import numpy as np

REL_STATE = 1e-5      # propagated / birth states: |d| <= 1e-5 max(|ref|, 1)
REL_C = 1e-4          # C entries and reweighted weights: rel 1e-4 ...
ABS_TINY = 1e-30      # ... or absolute 1e-30 for tiny values
GATE_BAND = 1e-4      # gate bits compared except where |L - gamma| <= 1e-4 gamma


def angdiff(a, b):
    return (np.asarray(a, np.float64) - np.asarray(b, np.float64) + math.pi) % (2 * math.pi) - math.pi


def check_state(gpu, ref, names=("x", "y", "v", "psi", "omega")):
    """gpu/ref: sequences of arrays in (x, y, v, psi, omega[, w]) order."""
    worst = {}
    for name, g, r in zip(names, gpu, ref):
        g = np.asarray(g, np.float64)
        r = np.asarray(r, np.float64)
        d = np.abs(angdiff(g, r)) if name == "psi" else np.abs(g - r)
        tol = REL_STATE * np.maximum(np.abs(r), 1.0)
        bad = d > tol
        assert not bad.any(), (f"{name}: {bad.sum()} entries off; worst d={d.max():.3e} "
                               f"at ref={r.ravel()[np.argmax(d)]:.6g}")
        worst[name] = float((d / np.maximum(np.abs(r), 1.0)).max()) if d.size else 0.0
    return worst


def unpack_gate(words, M):
    w = np.asarray(words).astype(np.uint32)
    bits = ((w[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    return bits.reshape(w.shape[0], -1)[:, :M]


def check_compat(gpu_C, gpu_gate, gpu_clutter, ref, gamma, M):
    """gpu_C [T, >=M] fp32, gpu_gate [T, >=ceil(M/32)] words; ref = oracle.compat dict.
    Returns (n_band, max_rel_err)."""
    T = ref["C_tracks"].shape[0]
    C = np.asarray(gpu_C, np.float64)[:T, :M]
    Lr = ref["L"]
    g32 = float(np.float32(gamma))
    band = np.abs(Lr - g32) <= GATE_BAND * g32
    ldg_used = (M + 31) // 32
    gbits = unpack_gate(np.asarray(gpu_gate)[:T, :ldg_used], M)
    rbits = unpack_gate(ref["gate"], M)
    mism = (gbits != rbits) & ~band
    assert not mism.any(), f"{mism.sum()} gate bits differ outside the gamma band"
    if M % 32:   # bits past M in the last word are zero
        last = np.asarray(gpu_gate)[:T, ldg_used - 1].astype(np.uint32)
        assert np.all((last >> np.uint32(M % 32)) == 0)
    Cr = ref["C_tracks"]
    d = np.abs(C - Cr)
    ok = (d <= REL_C * np.abs(Cr)) | (d <= ABS_TINY) | band
    assert ok.all(), (f"{(~ok).sum()} C entries off; worst rel "
                      f"{(d / np.maximum(np.abs(Cr), 1e-300))[~ok].max():.3e}")
    if gpu_clutter is not None:
        np.testing.assert_array_equal(np.asarray(gpu_clutter, np.float64)[:M], ref["C_clutter"])
    rel = d / np.maximum(np.abs(Cr), 1e-300)
    rel = rel[(Cr != 0) & ~band]
    return int(band.sum()), float(rel.max()) if rel.size else 0.0


def check_weights(gpu_w, ref_w):
    g = np.asarray(gpu_w, np.float64)
    r = np.asarray(ref_w, np.float64)
    d = np.abs(g - r)
    ok = (d <= REL_C * np.abs(r)) | (d <= ABS_TINY)
    assert ok.all(), f"{(~ok).sum()} weights off; worst d={d[~ok].max():.3e}"


def check_log_norm(gpu, ref):
    g = np.asarray(gpu, np.float64)
    r = np.asarray(ref, np.float64)
    same_inf = np.isinf(g) & np.isinf(r) & (np.sign(g) == np.sign(r))
    with np.errstate(invalid="ignore"):
        d = np.abs(g - r)
    ok = same_inf | (d <= REL_C * np.maximum(np.abs(r), 1.0))
    assert ok.all(), f"log_norm off: worst d={d[~ok].max():.3e}"
