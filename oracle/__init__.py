"""fp64 CPU oracle for the GLMB step core -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2512_06230_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``glmb_oracle.c`` (plain C, fp64, every
function cites the PAPER.md passage it follows); this module only builds it
with gcc and marshals numpy arrays through ctypes.

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
(see DESIGN.md "Oracle pins"); nothing is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "glmb_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile glmb_oracle.c -> oracle/liboracle.so (gcc -O2, OpenMP, no fast-math)."""
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
           "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB_PATH)
            P = np.ctypeslib.ndpointer
            f32 = P(np.float32, flags="C_CONTIGUOUS")
            f64 = P(np.float64, flags="C_CONTIGUOUS")
            i32 = P(np.int32, flags="C_CONTIGUOUS")
            u32 = P(np.uint32, flags="C_CONTIGUOUS")
            L.oracle_philox_batch.argtypes = [C.c_uint64, u32, C.c_int64, u32]
            L.oracle_uniform_u32.argtypes = [C.c_uint32]
            L.oracle_uniform_u32.restype = C.c_double
            L.oracle_normals4.argtypes = [C.c_uint64, u32, f64]
            L.oracle_normals_batch.argtypes = [C.c_uint64, u32, C.c_int64, f64]
            L.oracle_wrap.argtypes = [C.c_double]
            L.oracle_wrap.restype = C.c_double
            L.oracle_ctrv.argtypes = [f64, C.c_double, C.c_double, C.c_double, f64]
            L.oracle_gauss2.argtypes = [C.c_double] * 7
            L.oracle_gauss2.restype = C.c_double
            L.oracle_loggauss2.argtypes = [C.c_double] * 7
            L.oracle_loggauss2.restype = C.c_double
            L.oracle_predict.argtypes = (
                [C.c_int32, C.c_int32, C.c_int64] + [f32] * 5 + [i32]
                + [C.c_float] * 3 + [C.c_uint64, C.c_uint32] + [f64] * 5)
            L.oracle_birth.argtypes = (
                [C.c_int32, C.c_int32, C.c_int64, f32, f32, i32, C.c_uint64,
                 C.c_uint32] + [f64] * 6)
            L.oracle_compat.argtypes = (
                [C.c_int32, C.c_int32, C.c_int64, f32, f32, f32, C.c_int32, f32]
                + [C.c_float] * 6 + [f64, f64, f64, C.c_int64, u32, C.c_int64])
            L.oracle_reweight.argtypes = (
                [C.c_int32, C.c_int32, C.c_int64, f32, f32, f32, C.c_int32, f32]
                + [C.c_float] * 3 + [i32, C.c_int32, f64, f64, u32])
            u8 = P(np.uint8, flags="C_CONTIGUOUS")
            L.oracle_death_prob.argtypes = [C.c_int32, C.c_int32, f32, C.c_int64, u32, C.c_int64,
                                            C.c_float, C.c_float, f32, f64]
            L.oracle_compat_rows.argtypes = [C.c_int32, C.c_int32, f32, C.c_int64, u32, C.c_int64,
                                             i32, i32, f32, f64]
            L.oracle_assoc_sample.argtypes = (
                [C.c_int32] * 4 + [u32, C.c_int64, f64, f32, f32, C.c_float, C.c_float,
                                   i32, i32, f32, f64, f64, C.c_int32, C.c_uint64, C.c_uint32, u32, i32,
                                   C.c_int64, f64])
            L.oracle_dedup.argtypes = [C.c_int32] * 3 + [u32, C.c_int64, i32, C.c_int64, u8]
            L.oracle_prune.argtypes = [C.c_int32, f64, u8, C.c_double, C.c_int32, i32, f64]
            L.oracle_prune.restype = C.c_int32
            L.oracle_assoc_pairs.argtypes = [C.c_int32, i32, u32, C.c_int64, i32, C.c_int64, C.c_int32,
                                             C.c_int32, i32, i32, i32, i32]
            L.oracle_assoc_pairs.restype = C.c_int32
            L.oracle_reweight_pairs.argtypes = ([C.c_int32, C.c_int64, f32, f32, f32, f32]
                                                + [C.c_float] * 3 + [C.c_int32, i32, i32, i32, f64, f64, u32, f64])
            L.oracle_resample.argtypes = [C.c_int32, f32, C.c_uint64, C.c_uint32, C.c_int32, i32]
            L.oracle_resample.restype = C.c_int
            L.oracle_next_parents.argtypes = [C.c_int32, f64, i32, C.c_int32, C.c_int32, C.c_int32,
                                              C.c_int32, C.c_int64, u32, f64]
            L.oracle_map_estimate.argtypes = [C.c_int32, i32, C.c_int32, C.c_int32, C.c_int64, f32, f32,
                                              f32, f64]
            L.oracle_num_threads.restype = C.c_int
            L.oracle_set_num_threads.argtypes = [C.c_int]
            _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ----------------------------------------------------------------- O1-O4
def philox(seed: int, ctr: np.ndarray) -> np.ndarray:
    """Philox4x32-10 blocks for counters ctr [N,4] u32, key = (lo32, hi32)(seed)."""
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    out = np.empty_like(ctr)
    lib().oracle_philox_batch(C.c_uint64(seed), ctr, ctr.shape[0], out)
    return out


def uniform_u32(r: int) -> float:
    return float(lib().oracle_uniform_u32(int(r)))


def normals4(seed: int, ctr) -> np.ndarray:
    out = np.empty(4, np.float64)
    lib().oracle_normals4(C.c_uint64(seed), np.ascontiguousarray(ctr, np.uint32), out)
    return out


def normals_batch(seed: int, ctr: np.ndarray) -> np.ndarray:
    """Four normals per counter row (Box-Muller on words (0,1) and (2,3)) -> [N,4] fp64."""
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    out = np.empty(ctr.shape, np.float64)
    lib().oracle_normals_batch(C.c_uint64(seed), ctr, ctr.shape[0], out)
    return out


def wrap(a: float) -> float:
    return float(lib().oracle_wrap(float(a)))


# ----------------------------------------------------------------- O5
def ctrv(state, dt: float, nu_a: float = 0.0, nu_w: float = 0.0) -> np.ndarray:
    s = np.ascontiguousarray(state, np.float64)
    out = np.empty(5, np.float64)
    lib().oracle_ctrv(s, float(dt), float(nu_a), float(nu_w), out)
    return out


def predict(x, y, v, psi, omega, gid, dt, sigma_a, sigma_w, seed, step):
    """Arrays [T][ld] fp32; returns five fp64 arrays [T][ld] (P = ld)."""
    x, y, v, psi, omega = (_f32(a) for a in (x, y, v, psi, omega))
    T, ld = x.shape
    outs = [np.zeros((T, ld), np.float64) for _ in range(5)]
    lib().oracle_predict(T, ld, ld, x, y, v, psi, omega,
                         np.ascontiguousarray(gid, np.int32), float(dt),
                         float(sigma_a), float(sigma_w), C.c_uint64(seed),
                         C.c_uint32(step), *outs)
    return outs


# ----------------------------------------------------------------- O6
def birth(mean, chol, gid, P, seed, step):
    """mean [B,5], chol [B,15] fp32 -> six fp64 arrays [B][P] (x,y,v,psi,omega,w)."""
    mean, chol = _f32(mean), _f32(chol)
    B = mean.shape[0]
    outs = [np.zeros((B, P), np.float64) for _ in range(6)]
    lib().oracle_birth(B, P, P, mean, chol, np.ascontiguousarray(gid, np.int32),
                       C.c_uint64(seed), C.c_uint32(step), *outs)
    return outs


# ----------------------------------------------------------------- O7
def gauss2(z, p, R) -> float:
    return float(lib().oracle_gauss2(float(z[0]), float(z[1]), float(p[0]), float(p[1]),
                                     float(R[0]), float(R[1]), float(R[2])))


def loggauss2(z, p, R) -> float:
    return float(lib().oracle_loggauss2(float(z[0]), float(z[1]), float(p[0]), float(p[1]),
                                        float(R[0]), float(R[1]), float(R[2])))


def compat(x, y, w, Z, R, p_d, kappa, gamma):
    """x,y,w [T][P] fp32, Z [M,2] fp32, R = (Rxx,Rxy,Ryy).
    Returns dict: L [T][M] (no P_D), C_clutter [M], C_tracks [T][M], gate [T][ceil(M/32)]."""
    x, y, w = (_f32(a).reshape(np.shape(a)[0], -1) if np.size(a) else
               np.zeros((np.shape(a)[0] if np.ndim(a) else 0, 4), np.float32) for a in (x, y, w))
    Z = _f32(Z).reshape(-1, 2)
    T, P = x.shape
    M = Z.shape[0]
    ldg = (M + 31) // 32
    Lik = np.zeros((T, M), np.float64)
    Ccl = np.zeros(M, np.float64)
    Ctr = np.zeros((T, M), np.float64)
    gate = np.zeros((T, ldg), np.uint32)
    lib().oracle_compat(T, P, P, x, y, w, M, Z, float(R[0]), float(R[1]), float(R[2]),
                        float(p_d), float(kappa), float(gamma), Lik, Ccl, Ctr, M, gate, ldg)
    return {"L": Lik, "C_clutter": Ccl, "C_tracks": Ctr, "gate": gate}


# ----------------------------------------------------------------- O8
def reweight(x, y, w, Z, R, theta, col_offset=0):
    """Returns (w' [T][P] fp64, logZ [T] fp64, flags [T] u32)."""
    x, y, w = _f32(x), _f32(y), _f32(w)
    Z = _f32(Z).reshape(-1, 2)
    T, P = x.shape
    M = Z.shape[0]
    wo = np.zeros((T, P), np.float64)
    lz = np.zeros(T, np.float64)
    fl = np.zeros(T, np.uint32)
    lib().oracle_reweight(T, P, P, x, y, w, M, Z, float(R[0]), float(R[1]), float(R[2]),
                          np.ascontiguousarray(theta, np.int32), int(col_offset), wo, lz, fl)
    return wo, lz, fl


def nearest_gate_theta(ref_compat) -> np.ndarray:
    """Nearest-gate association map of BASELINE.json configs[2] ("A nearest-gate association map
    theta is supplied for reweighting each step"), computed from the ORACLE's C_k (a dict returned
    by ``compat``): theta_i = 1 + argmax_j {C[i, j+1] : g_ij = 1} (ties -> lowest j), 0 when row i
    has no gated track (the clutter column).  Test/bench harness input (reading R22)."""
    C = np.asarray(ref_compat["C_tracks"], np.float64)       # [T][M]
    T, M = C.shape
    if T == 0 or M == 0:
        return np.zeros(M, np.int32)
    g = ((np.asarray(ref_compat["gate"], np.uint32)[:, np.arange(M) // 32]
          >> (np.arange(M) % 32).astype(np.uint32)) & 1).astype(bool)      # [T][M]
    Cg = np.where(g, C, -np.inf)
    j = np.argmax(Cg, axis=0)                                  # first maximiser = lowest j
    return np.where(g.any(axis=0), j + 1, 0).astype(np.int32)


# ----------------------------------------------------------------- O9-O13 (hypothesis machinery)
def _gate_words(gate, T, M):
    ldg = (M + 31) // 32
    if T == 0:
        return np.zeros((1, 1), np.uint32), ldg
    g = np.ascontiguousarray(gate, np.uint32).reshape(T, -1)
    return g, g.shape[1]


def death_prob(C_tracks, gate, p_d, kappa, p_s):
    """C_tracks fp32 [T][ldc] (column-major C), gate u32 [T][ldg]; p_s [T] -> d [T] fp64 (O9)."""
    C = _f32(C_tracks)
    T = C.shape[0]
    ldc = C.shape[1] if T else 0
    g, ldg = _gate_words(gate, T, ldc)
    M = ldc
    d = np.zeros(T, np.float64)
    lib().oracle_death_prob(T, M, C, ldc, g, ldg, float(p_d), float(kappa), _f32(p_s), d)
    return d


def compat_rows(C_tracks, gate, M):
    """Row-wise (CSR) view of C: (row_ptr [M+1] i32, col [nnz] i32, val [nnz] f32, ln_val [nnz] f64) (O10)."""
    C = _f32(C_tracks)
    T = C.shape[0]
    ldc = C.shape[1] if T else M
    g, ldg = _gate_words(gate, T, M)
    cap = max(1, T * M)
    rp = np.zeros(M + 1, np.int32)
    col = np.zeros(cap, np.int32)
    val = np.zeros(cap, np.float32)
    lv = np.zeros(cap, np.float64)
    lib().oracle_compat_rows(T, M, C if T else np.zeros((1, 1), np.float32), ldc,
                             g if T else np.zeros((1, 1), np.uint32), ldg, rp, col, val, lv)
    n = int(rp[M])
    return rp, col[:n].copy(), val[:n].copy(), lv[:n].copy()


def assoc_sample(parent_mask, parent_logw, H_up, d_prob, p_s, p_d, kappa, rows, M, seed, step,
                 count_lp=None):
    """Two-stage sampler (O11).  parent_mask u32 [H_old][ldt]; rows = compat_rows(...);
    count_lp: optional ln prior of the number of measurements per alive track (index min(n, len-1)).
    Returns (alive u32 [H_old*H_up][ldt], theta i32 [H_old*H_up][M], logw f64 [H_old*H_up])."""
    clp = np.ascontiguousarray(count_lp if count_lp is not None else np.zeros(1), np.float64)
    n_count = 0 if count_lp is None else len(clp)
    pm = np.ascontiguousarray(parent_mask, np.uint32)
    H_old, ldt = pm.shape
    T = len(d_prob)
    rp, col, val, lv = rows
    n = H_old * H_up
    alive = np.zeros((n, ldt), np.uint32)
    theta = np.zeros((n, max(M, 1)), np.int32)
    logw = np.zeros(n, np.float64)
    one = lambda a, dt: np.ascontiguousarray(a if len(a) else np.zeros(1, dt), dt)
    lib().oracle_assoc_sample(H_old, H_up, T, M, pm, ldt, np.ascontiguousarray(parent_logw, np.float64),
                              one(d_prob, np.float32), one(p_s, np.float32), float(p_d), float(kappa),
                              np.ascontiguousarray(rp, np.int32), one(col, np.int32), one(val, np.float32),
                              one(lv, np.float64), clp, n_count, C.c_uint64(seed), C.c_uint32(step),
                              alive, theta,
                              theta.shape[1], logw)
    return alive, theta[:, :M], logw


def dedup(alive, theta, H_old, H_up):
    """unique u8 [H_old*H_up]: 1 for the first occurrence of each (alive, theta) within a parent (O12)."""
    al = np.ascontiguousarray(alive, np.uint32)
    th = np.ascontiguousarray(theta, np.int32)
    M = th.shape[1]
    if M == 0:
        th = np.zeros((th.shape[0], 1), np.int32)
    u = np.zeros(H_old * H_up, np.uint8)
    lib().oracle_dedup(H_old, H_up, M, al, al.shape[1], th, th.shape[1], u)
    return u


def prune(logw, unique, tau, h_max):
    """(keep_idx i32 [k], keep_w f64 [k]) after normalisation, tau and H_max (O13)."""
    lw = np.ascontiguousarray(logw, np.float64)
    u = np.ascontiguousarray(unique, np.uint8)
    n = len(lw)
    idx = np.zeros(max(1, n), np.int32)
    w = np.zeros(max(1, n), np.float64)
    k = lib().oracle_prune(n, lw if n else np.zeros(1), u if n else np.zeros(1, np.uint8),
                           float(tau), int(h_max), idx, w)
    return idx[:k].copy(), w[:k].copy()


# ----------------------------------------------------------------- O14-O16 (particle loop)
def assoc_pairs(hyp_idx, alive, theta, T, M):
    """Unique (track, measurement-set) pairs over the hypotheses hyp_idx (O14).
    Returns (pair_track [K], pair_ptr [K+1], pair_meas [nnz], pair_of [n_hyp][T])."""
    hi = np.ascontiguousarray(hyp_idx, np.int32)
    al = np.ascontiguousarray(alive, np.uint32)
    th = np.ascontiguousarray(theta, np.int32)
    if th.shape[1] == 0:
        th = np.zeros((th.shape[0], 1), np.int32)
    n = len(hi)
    cap = max(1, n * T)
    pt = np.zeros(cap, np.int32)
    pp = np.zeros(cap + 1, np.int32)
    pm = np.zeros(max(1, n * M), np.int32)
    po = np.zeros((max(n, 1), max(T, 1)), np.int32)
    K = lib().oracle_assoc_pairs(n, hi if n else np.zeros(1, np.int32), al, al.shape[1], th, th.shape[1],
                                 T, M, pt, pp, pm, po)
    return pt[:K].copy(), pp[:K + 1].copy(), pm[:pp[K]].copy(), po[:n, :T].copy()


def reweight_pairs(x, y, w, Z, R, pair_track, pair_ptr, pair_meas):
    """Per-pair Bayes update (O15): (w' [K][P] fp64, logZ [K], flags [K] u32, ess [K])."""
    x, y, w = _f32(x), _f32(y), _f32(w)
    Z = _f32(Z).reshape(-1, 2)
    if Z.shape[0] == 0:
        Z = np.zeros((1, 2), np.float32)
    P = x.shape[1]
    K = len(pair_track)
    wo = np.zeros((max(K, 1), P), np.float64)
    lz = np.zeros(max(K, 1), np.float64)
    fl = np.zeros(max(K, 1), np.uint32)
    es = np.zeros(max(K, 1), np.float64)
    pm = np.ascontiguousarray(pair_meas, np.int32)
    lib().oracle_reweight_pairs(P, P, x, y, w, Z, float(R[0]), float(R[1]), float(R[2]), K,
                                np.ascontiguousarray(pair_track if K else np.zeros(1), np.int32),
                                np.ascontiguousarray(pair_ptr, np.int32),
                                pm if len(pm) else np.zeros(1, np.int32), wo, lz, fl, es)
    return wo[:K], lz[:K], fl[:K], es[:K]


def resample(w, seed, step, k):
    """Systematic resampling decision + ancestors of one weight vector (O16): (resampled, anc [P])."""
    w = _f32(w)
    anc = np.full(len(w), -1, np.int32)
    r = lib().oracle_resample(len(w), w, C.c_uint64(seed), C.c_uint32(step), int(k), anc)
    return bool(r), anc


# ----------------------------------------------------------------- O17-O18 (tracker loop)
def next_parents(keep_w, pair_of, T, K_cap, B, birth_col0, ldt):
    """(mask u32 [n_kept][ldt], logw f64 [n_kept]) of the next step's parents (O17)."""
    kw = np.ascontiguousarray(keep_w, np.float64)
    n = len(kw)
    po = np.ascontiguousarray(pair_of, np.int32).reshape(max(n, 1), -1) if n else np.zeros((1, max(T, 1)), np.int32)
    mask = np.zeros((max(n, 1), ldt), np.uint32)
    lw = np.zeros(max(n, 1), np.float64)
    lib().oracle_next_parents(n, kw if n else np.zeros(1), po, T, K_cap, B, birth_col0, ldt, mask, lw)
    return mask[:n], lw[:n]


def map_estimate(n_kept, pair_of0, x, y, w):
    """est [T][3] = (x, y, 1) weighted mean of row pair_of0[j] of (x, y, w), or (nan, nan, 0) (O18)."""
    x, y, w = _f32(x), _f32(y), _f32(w)
    po = np.ascontiguousarray(pair_of0, np.int32)
    T = len(po)
    P = x.shape[1]
    est = np.zeros((max(T, 1), 3), np.float64)
    lib().oracle_map_estimate(int(n_kept), po if T else np.zeros(1, np.int32), T, P, P, x, y, w, est)
    return est[:T]
