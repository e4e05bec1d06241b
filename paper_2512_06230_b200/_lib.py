"""Thin ctypes binding of libglmb.so (include/glmb.h).  Argument marshalling only.

Every function here has the name of the C entry point it calls and takes
torch CUDA tensors (device memory allocated by torch) plus an optional
``torch.cuda.Stream``.  No arithmetic of the method happens in Python, and
there is no CPU fallback: if the library is missing or the device is not
sm_100a, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GLMB_LIB", os.path.join(_HERE, "libglmb.so"))  # override: A/B runs only

GLMB_OK = 0
_lock = threading.Lock()
_lib = None


class GlmbError(RuntimeError):
    def __init__(self, status: int, text: str):
        super().__init__(f"{text} (status {status})")
        self.status = status


class glmb_particles(C.Structure):
    _fields_ = [("x", C.c_void_p), ("y", C.c_void_p), ("v", C.c_void_p), ("psi", C.c_void_p),
                ("omega", C.c_void_p), ("w", C.c_void_p), ("n_tracks", C.c_int32),
                ("n_particles", C.c_int32), ("ld", C.c_int64)]


class glmb_step_params(C.Structure):
    _fields_ = [("tracks", glmb_particles), ("n_survivors", C.c_int32), ("gid", C.c_void_p),
                ("birth_mean", C.c_void_p), ("birth_chol", C.c_void_p), ("dt", C.c_float),
                ("sigma_a", C.c_float), ("sigma_w", C.c_float), ("seed", C.c_uint64),
                ("step", C.c_uint32), ("Rxx", C.c_float), ("Rxy", C.c_float), ("Ryy", C.c_float),
                ("p_d", C.c_float), ("kappa", C.c_float), ("gamma", C.c_float),
                ("col_offset", C.c_int32), ("w_out", C.c_void_p)]


class glmb_update_params(C.Structure):
    vp, i32, i64, f32, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double
    _fields_ = [("T", i32), ("M", i32), ("H_old", i32), ("H_up", i32), ("h_max", i32), ("K_cap", i32),
                ("p_d", f32), ("kappa", f32), ("Rxx", f32), ("Rxy", f32), ("Ryy", f32), ("tau", f64),
                ("seed", C.c_uint64), ("step", C.c_uint32), ("tracks", glmb_particles),
                ("C_tracks", vp), ("ldc", i64), ("gate", vp), ("ldg", i64), ("Z", vp), ("p_s", vp),
                ("parent_mask", vp), ("ldt", i32), ("parent_logw", vp), ("n_parents", vp), ("count_lp", vp),
                ("n_count", i32), ("d_prob", vp), ("row_ptr", vp), ("col", vp), ("val", vp), ("ln_val", vp),
                ("rows_cap", i32), ("alive", vp), ("theta", vp), ("ldm", i64), ("logw", vp), ("hash", vp),
                ("unique", vp), ("prune_ws", vp), ("keep_idx", vp), ("keep_w", vp), ("n_kept", vp),
                ("pair_track", vp), ("pair_ptr", vp), ("pair_meas", vp), ("pair_of", vp), ("n_pairs", vp),
                ("pairs_ws", vp), ("pairs_ws_bytes", C.c_size_t), ("w_new", vp), ("ld_new", i64),
                ("log_norm", vp), ("flags", vp), ("ess", vp), ("out", glmb_particles), ("est", vp)]


EXPORTED = ["glmb_version", "glmb_status_string", "glmb_init", "glmb_sm_count", "glmb_predict",
            "glmb_birth", "glmb_compat", "glmb_reweight", "glmb_step", "glmb_step_host",
            "glmb_philox_dump", "glmb_normals_dump", "glmb_death_prob", "glmb_compat_rows",
            "glmb_assoc_sample", "glmb_dedup", "glmb_prune", "glmb_assoc_pairs_workspace_size",
            "glmb_assoc_pairs", "glmb_reweight_pairs", "glmb_resample", "glmb_next_parents",
            "glmb_map_estimate", "glmb_update", "glmb_compat_peers", "glmb_step_host_csr", "glmb_compat_skipping"]


def load(path: str = LIB_PATH):
    """dlopen libglmb.so and declare every signature.  Raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise GlmbError(-100, f"libglmb.so not built at {path}: run "
                                  f"`python -m paper_2512_06230_b200.build` (no CPU fallback exists)")
        L = C.CDLL(path)
        vp, i32, i64, u32, u64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float
        PP = C.POINTER(glmb_particles)
        L.glmb_version.restype = C.c_int
        L.glmb_status_string.restype = C.c_char_p
        L.glmb_status_string.argtypes = [C.c_int]
        L.glmb_init.argtypes = [C.c_int]
        L.glmb_sm_count.argtypes = [C.c_int]
        L.glmb_predict.argtypes = [PP, PP, vp, f32, f32, f32, u64, u32, vp]
        L.glmb_birth.argtypes = [PP, vp, vp, vp, u64, u32, vp]
        L.glmb_compat.argtypes = [PP, vp, i32, f32, f32, f32, f32, f32, f32, vp, vp, i64, vp, i64, vp]
        L.glmb_compat_skipping.argtypes = [PP, vp, i32, f32, f32, f32, f32, f32, f32, vp, vp, i64, vp, i64, vp, vp]
        L.glmb_reweight.argtypes = [PP, vp, vp, i32, f32, f32, f32, vp, i32, vp, vp, vp]
        SP = C.POINTER(glmb_step_params)
        L.glmb_step.argtypes = [SP, vp, i32, vp, vp, vp, i64, vp, i64, vp, vp, vp]
        L.glmb_step_host.argtypes = [SP, vp, i32, vp, vp, vp, vp, vp, i64, vp, i64, vp, vp,
                                     vp, vp, vp, vp, vp, vp, vp]
        L.glmb_philox_dump.argtypes = [u64, vp, i32, vp, vp]
        L.glmb_normals_dump.argtypes = [u64, vp, i32, vp, vp]
        L.glmb_death_prob.argtypes = [i32, i32, vp, i64, vp, i64, f32, f32, vp, vp, vp]
        L.glmb_compat_rows.argtypes = [i32, i32, vp, i64, vp, i64, vp, vp, vp, vp, i32, vp]
        L.glmb_assoc_sample.argtypes = [i32, vp, i32, i32, i32, vp, i32, vp, vp, vp, f32, f32, vp, vp, vp,
                                        vp, vp, i32, u64, u32, vp, vp, i64, vp, vp, vp]
        L.glmb_dedup.argtypes = [i32, vp, i32, i32, vp, i32, vp, i64, vp, vp, vp]
        L.glmb_next_parents.argtypes = [i32, vp, vp, vp, i32, i32, i32, i32, vp, i32, vp, vp, vp, vp]
        L.glmb_map_estimate.argtypes = [vp, vp, i32, PP, vp, vp]
        L.glmb_update.argtypes = [C.POINTER(glmb_update_params), vp]
        L.glmb_step_host_csr.argtypes = [SP, vp, i32, vp, vp, vp, vp, i64, vp, i64, vp, vp, vp, vp, vp, vp,
                                         i32, vp, vp, vp, i32, i32, vp, vp, vp, vp]
        L.glmb_compat_peers.argtypes = [PP, vp, i32, f32, f32, f32, f32, f32, f32, vp, vp, vp, i32, i64, i64,
                                        i64, vp]
        L.glmb_prune.argtypes = [i32, vp, vp, C.c_double, i32, vp, vp, vp, vp, vp]
        L.glmb_assoc_pairs_workspace_size.argtypes = [i32, i32, i32]
        L.glmb_assoc_pairs_workspace_size.restype = C.c_size_t
        L.glmb_assoc_pairs.argtypes = [i32, vp, vp, vp, i32, vp, i64, i32, i32, vp, vp, vp, vp, vp, vp,
                                       C.c_size_t, vp]
        L.glmb_reweight_pairs.argtypes = [PP, vp, i32, f32, f32, f32, i32, vp, vp, vp, vp, vp, i64, vp, vp,
                                          vp, vp]
        L.glmb_resample.argtypes = [PP, i32, vp, vp, vp, i64, PP, u64, u32, vp, vp]
        for name in EXPORTED:
            if name not in ("glmb_version", "glmb_status_string", "glmb_sm_count",
                            "glmb_assoc_pairs_workspace_size"):
                getattr(L, name).restype = C.c_int
        _lib = L
        return L


def _check(status: int) -> None:
    if status != GLMB_OK:
        raise GlmbError(status, load().glmb_status_string(status).decode())


def _ptr(t) -> int:
    if t is None:
        return None
    if not t.is_cuda:
        raise GlmbError(-1, "expected a CUDA tensor (the GLMB path has no CPU fallback)")
    if not t.is_contiguous():
        raise GlmbError(-1, "expected a contiguous tensor")
    return t.data_ptr()


def _mat(t):
    """(pointer, leading dimension) of a row-major 2-D CUDA matrix whose rows may be strided
    (e.g. the C columns / gate words of a packed row, dist.ShardedStep); None -> (None, 0)."""
    if t is None:
        return None, 0
    if not t.is_cuda:
        raise GlmbError(-1, "expected a CUDA tensor (the GLMB path has no CPU fallback)")
    if t.dim() != 2:
        raise GlmbError(-1, "expected a 2-D matrix")
    if t.numel() == 0 or t.shape[0] == 1:
        return t.data_ptr(), t.shape[1]
    if t.shape[1] > 1 and t.stride(1) != 1:
        raise GlmbError(-1, "expected a 2-D matrix with unit column stride")
    return t.data_ptr(), t.stride(0)


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Particles:
    """SoA particle storage: one tensor [6, T, ld] fp32 (x, y, v, psi, omega, w)."""

    FIELDS = ("x", "y", "v", "psi", "omega", "w")

    def __init__(self, data: torch.Tensor, n_particles: int, w: torch.Tensor | None = None):
        """w: optional separate weight buffer [T, ld] used instead of data[5]."""
        assert data.dim() == 3 and data.shape[0] == 6 and data.dtype == torch.float32
        self.data = data
        self.T = data.shape[1]
        self.ld = data.shape[2]
        self.P = n_particles
        self.w_override = w

    @classmethod
    def empty(cls, T: int, P: int, device="cuda", ld: int | None = None):
        ld = P if ld is None else ld
        return cls(torch.empty(6, T, ld, dtype=torch.float32, device=device), P)

    @classmethod
    def from_arrays(cls, arrays, device="cuda"):
        """arrays: six [T, P] array-likes (x, y, v, psi, omega, w)."""
        t = torch.stack([torch.as_tensor(a, dtype=torch.float32) for a in arrays]).contiguous()
        return cls(t.to(device), t.shape[2])

    def rows(self, start: int, stop: int) -> "Particles":
        w = None if self.w_override is None else self.w_override[start:stop]
        return Particles(self.data[:, start:stop], self.P, w)

    def weights(self) -> torch.Tensor:
        return self.data[5] if self.w_override is None else self.w_override

    def field(self, name: str) -> torch.Tensor:
        return self.data[self.FIELDS.index(name)]

    def struct(self) -> glmb_particles:
        d = self.data
        T = d.shape[1]
        if T == 0:
            return glmb_particles(None, None, None, None, None, None, 0, self.P, self.ld)
        if d.stride(2) != 1 or d.stride(1) != self.ld:
            raise GlmbError(-1, "particle storage must be [6][T][ld] with unit stride")
        if not d.is_cuda:
            raise GlmbError(-1, "particles must live in CUDA memory")
        base, fs = d.data_ptr(), d.stride(0) * 4   # field k at base + k * fs bytes
        ptrs = [base + k * fs for k in range(6)]
        if self.w_override is not None:
            ptrs[5] = self.w_override.data_ptr()
        return glmb_particles(*ptrs, T, self.P, self.ld)


# --------------------------------------------------------------- entry points
def glmb_version() -> int:
    return load().glmb_version()


def glmb_init(device: int = 0) -> None:
    _check(load().glmb_init(device))


def glmb_sm_count(device: int = 0) -> int:
    return load().glmb_sm_count(device)


def glmb_predict(inp: Particles, out: Particles, gid, dt, sigma_a, sigma_w, seed, step, stream=None):
    a, b = inp.struct(), out.struct()
    _check(load().glmb_predict(C.byref(a), C.byref(b), _ptr(gid), dt, sigma_a, sigma_w,
                               int(seed) & 0xFFFFFFFFFFFFFFFF, int(step), _stream(stream)))


def glmb_birth(out: Particles, gid, mean, chol, seed, step, stream=None):
    b = out.struct()
    _check(load().glmb_birth(C.byref(b), _ptr(gid), _ptr(mean), _ptr(chol),
                             int(seed) & 0xFFFFFFFFFFFFFFFF, int(step), _stream(stream)))


def glmb_compat(trk: Particles, Z, R, p_d, kappa, gamma, C_clutter, C_tracks, gate, stream=None):
    """Z [M,2] fp32; C_tracks [T, ldc] fp32; gate [T, ldg] int32 (u32 words); C_clutter [M] or None."""
    t = trk.struct()
    M = Z.shape[0]
    (pc, ldc), (pg, ldg) = _mat(C_tracks), _mat(gate)
    _check(load().glmb_compat(C.byref(t), _ptr(Z), M, R[0], R[1], R[2], p_d, kappa, gamma,
                              _ptr(C_clutter), pc, ldc, pg, ldg, _stream(stream)))


def glmb_compat_skipping(trk: Particles, Z, R, p_d, kappa, gamma, C_clutter, C_tracks, gate, skipped=None,
                         stream=None):
    """glmb_compat with exact zero-tile skipping (include/glmb.h); skipped: optional device uint64 [1]
    (int64 tensor) incremented by the number of skipped pairs."""
    t = trk.struct()
    M = Z.shape[0]
    (pc, ldc), (pg, ldg) = _mat(C_tracks), _mat(gate)
    _check(load().glmb_compat_skipping(C.byref(t), _ptr(Z), M, R[0], R[1], R[2], p_d, kappa, gamma,
                                       _ptr(C_clutter), pc, ldc, pg, ldg, _ptr(skipped), _stream(stream)))


def glmb_reweight(trk: Particles, Z, R, theta, col_offset, log_norm, flags, stream=None, w_out=None):
    """w_out: [T, ld] tensor for the new weights (None: in place, trk's w)."""
    t = trk.struct()
    wo = t.w if w_out is None else _ptr(w_out)
    _check(load().glmb_reweight(C.byref(t), wo, _ptr(Z), Z.shape[0], R[0], R[1], R[2], _ptr(theta),
                                int(col_offset), _ptr(log_norm), _ptr(flags), _stream(stream)))


def make_step_params(tracks: Particles, n_survivors, gid, birth_mean, birth_chol, dt, sigma_a,
                     sigma_w, seed, step, R, p_d, kappa, gamma, col_offset=0, w_out=None) -> glmb_step_params:
    """w_out: optional spare weight buffer [T_k, ld] for the new weights (see glmb.h)."""
    return glmb_step_params(tracks.struct(), int(n_survivors), _ptr(gid), _ptr(birth_mean),
                            _ptr(birth_chol), dt, sigma_a, sigma_w, int(seed) & 0xFFFFFFFFFFFFFFFF,
                            int(step), R[0], R[1], R[2], p_d, kappa, gamma, int(col_offset), _ptr(w_out))


def glmb_step(prm: glmb_step_params, Z, theta, C_clutter, C_tracks, gate, log_norm, flags,
              stream=None):
    _check(load().glmb_step(C.byref(prm), _ptr(Z), Z.shape[0], _ptr(theta), _ptr(C_clutter),
                            _ptr(C_tracks), C_tracks.shape[1], _ptr(gate), gate.shape[1],
                            _ptr(log_norm), _ptr(flags), _stream(stream)))


def glmb_step_host(prm: glmb_step_params, Z_host, theta_host, Z_dev, theta_dev, C_clutter,
                   C_tracks, gate, log_norm, flags, C_clutter_host, C_tracks_host, gate_host,
                   log_norm_host, flags_host, stream=None, copy_stream=None):
    """Host tensors (pinned recommended) in and out; synchronous.  copy_stream: a second
    torch.cuda.Stream for the overlapped read-back (see glmb.h)."""
    hp = lambda t: None if t is None else t.data_ptr()
    M = Z_host.shape[0]
    _check(load().glmb_step_host(C.byref(prm), hp(Z_host), M, hp(theta_host), _ptr(Z_dev),
                                 _ptr(theta_dev), _ptr(C_clutter), _ptr(C_tracks), C_tracks.shape[1],
                                 _ptr(gate), gate.shape[1], _ptr(log_norm), _ptr(flags),
                                 hp(C_clutter_host), hp(C_tracks_host), hp(gate_host),
                                 hp(log_norm_host), hp(flags_host), _stream(stream),
                                 None if copy_stream is None else copy_stream.cuda_stream))


def glmb_philox_dump(seed, ctr, out, stream=None):
    _check(load().glmb_philox_dump(int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(ctr), ctr.shape[0],
                                   _ptr(out), _stream(stream)))


def glmb_normals_dump(seed, ctr, out, stream=None):
    _check(load().glmb_normals_dump(int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(ctr), ctr.shape[0],
                                    _ptr(out), _stream(stream)))


# --------------------------------------------------------------- hypothesis machinery (f1, f3)
def glmb_death_prob(C_tracks, gate, M, p_d, kappa, p_s, d_out, stream=None):
    """C_tracks [T, ldc] fp32, gate [T, ldg] int32 words, p_s [T] fp32 -> d_out [T] fp32."""
    T = C_tracks.shape[0]
    (pc, ldc), (pg, ldg) = _mat(C_tracks), _mat(gate)
    _check(load().glmb_death_prob(T, int(M), pc, ldc, pg, ldg, p_d, kappa, _ptr(p_s), _ptr(d_out),
                                  _stream(stream)))


def glmb_compat_rows(C_tracks, gate, M, row_ptr, col, val, ln_val, stream=None):
    """CSR of the gated entries: row_ptr [M+1] int32, col [cap] int32, val [cap] fp32, ln_val [cap] fp64."""
    T = C_tracks.shape[0]
    (pc, ldc), (pg, ldg) = _mat(C_tracks), _mat(gate)
    _check(load().glmb_compat_rows(T, int(M), pc, ldc, pg, ldg, _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(ln_val), col.shape[0],
                                   _stream(stream)))


def glmb_assoc_sample(H_up, parent_mask, parent_logw, d_prob, p_s, p_d, kappa, row_ptr, col, val, ln_val,
                      M, seed, step, alive, theta, logw, hash=None, stream=None, n_parents=None,
                      count_lp=None):
    """parent_mask [H_old, ldt] int32 words; alive [H_old*H_up, ldt]; theta [H_old*H_up, ldm] int32.
    n_parents: optional device int32 count of valid parent rows."""
    H_old, ldt = parent_mask.shape
    T = d_prob.shape[0]
    _check(load().glmb_assoc_sample(H_old, _ptr(n_parents), int(H_up), T, int(M), _ptr(parent_mask), ldt, _ptr(parent_logw),
                                    _ptr(d_prob), _ptr(p_s), p_d, kappa, _ptr(row_ptr), _ptr(col), _ptr(val),
                                    _ptr(ln_val), _ptr(count_lp), 0 if count_lp is None else count_lp.shape[0],
                                    int(seed) & 0xFFFFFFFFFFFFFFFF, int(step), _ptr(alive),
                                    _ptr(theta), theta.shape[1], _ptr(logw), _ptr(hash), _stream(stream)))


def glmb_dedup(H_old, H_up, M, alive, theta, hash, unique, stream=None, n_parents=None):
    _check(load().glmb_dedup(int(H_old), _ptr(n_parents), int(H_up), int(M), _ptr(alive), alive.shape[1], _ptr(theta),
                             theta.shape[1], _ptr(hash), _ptr(unique), _stream(stream)))


def glmb_prune(logw, unique, tau, h_max, workspace, keep_idx, keep_w, n_kept, stream=None):
    _check(load().glmb_prune(logw.shape[0], _ptr(logw), _ptr(unique), float(tau), int(h_max), _ptr(workspace),
                             _ptr(keep_idx), _ptr(keep_w), _ptr(n_kept), _stream(stream)))


# --------------------------------------------------------------- particle loop (f2)
def glmb_assoc_pairs_workspace_size(n_hyp, T, M) -> int:
    return int(load().glmb_assoc_pairs_workspace_size(int(n_hyp), int(T), int(M)))


def glmb_assoc_pairs(hyp_idx, alive, theta, T, M, pair_track, pair_ptr, pair_meas, pair_of, n_pairs,
                     workspace, stream=None, n_hyp_dev=None):
    """hyp_idx [n_hyp] int32 rows of alive [., ldt] / theta [., ldm]; outputs as in glmb.h.
    n_hyp_dev: optional device int32 count of hypotheses actually used (e.g. glmb_prune's n_kept)."""
    n_hyp = hyp_idx.shape[0]
    _check(load().glmb_assoc_pairs(n_hyp, _ptr(n_hyp_dev), _ptr(hyp_idx), _ptr(alive), alive.shape[1], _ptr(theta),
                                   theta.shape[1], int(T), int(M), _ptr(pair_track), _ptr(pair_ptr),
                                   _ptr(pair_meas), _ptr(pair_of), _ptr(n_pairs), _ptr(workspace),
                                   workspace.numel() * workspace.element_size(), _stream(stream)))


def glmb_reweight_pairs(src: Particles, Z, R, K, n_pairs, pair_track, pair_ptr, pair_meas, w_out, log_norm,
                        flags, ess, stream=None):
    t = src.struct()
    _check(load().glmb_reweight_pairs(C.byref(t), _ptr(Z), Z.shape[0], R[0], R[1], R[2], int(K), _ptr(n_pairs),
                                      _ptr(pair_track), _ptr(pair_ptr), _ptr(pair_meas), _ptr(w_out),
                                      w_out.shape[1], _ptr(log_norm), _ptr(flags), _ptr(ess), _stream(stream)))


def glmb_resample(src: Particles, K, n_pairs, pair_track, w, out: Particles, seed, step, flags=None,
                  stream=None):
    a, b = src.struct(), out.struct()
    _check(load().glmb_resample(C.byref(a), int(K), _ptr(n_pairs), _ptr(pair_track), _ptr(w), w.shape[1],
                                C.byref(b), int(seed) & 0xFFFFFFFFFFFFFFFF, int(step), _ptr(flags),
                                _stream(stream)))


# --------------------------------------------------------------- tracker loop (f4)
def glmb_next_parents(n_kept, keep_w, pair_of, K_cap, B, birth_col0, parent_mask, parent_logw, n_parents,
                      stream=None, birth_col0_dev=None):
    """pair_of [n_hyp_cap, T] int32; parent_mask [n_hyp_cap, ldt] int32 words (outputs on device).
    birth_col0_dev: optional device int32 (e.g. n_pairs) overriding birth_col0."""
    n_hyp_cap, T = pair_of.shape
    _check(load().glmb_next_parents(n_hyp_cap, _ptr(n_kept), _ptr(keep_w), _ptr(pair_of), T, int(K_cap), int(B),
                                    int(birth_col0), _ptr(parent_mask), parent_mask.shape[1], _ptr(parent_logw),
                                    _ptr(n_parents), _ptr(birth_col0_dev), _stream(stream)))


def glmb_map_estimate(n_kept, pair_of0, new_set: Particles, est, stream=None):
    """pair_of0 [T] int32 (row 0 of pair_of); est [T, 3] fp64."""
    t = new_set.struct()
    _check(load().glmb_map_estimate(_ptr(n_kept), _ptr(pair_of0), pair_of0.shape[0], C.byref(t), _ptr(est),
                                    _stream(stream)))


def glmb_update(params: "glmb_update_params", stream=None):
    """The whole update after C_k in one C call (include/glmb.h glmb_update)."""
    _check(load().glmb_update(C.byref(params), _stream(stream)))


def glmb_compat_peers(trk: Particles, Z, R, p_d, kappa, gamma, C_clutter, peer_C, peer_G, row0, ldc, ldg,
                      stream=None):
    """Fused compat + all-gather: peer_C / peer_G are device int64 tensors [n_peers] of device pointers
    (e.g. torch symmetric memory's buffer_ptrs_dev); column j goes to row row0 + j of every peer."""
    t = trk.struct()
    _check(load().glmb_compat_peers(C.byref(t), _ptr(Z), Z.shape[0], R[0], R[1], R[2], p_d, kappa, gamma,
                                    _ptr(C_clutter), _ptr(peer_C), _ptr(peer_G), peer_C.shape[0], int(row0),
                                    int(ldc), int(ldg), _stream(stream)))


def glmb_step_host_csr(prm: glmb_step_params, Z_host, theta_host, Z_dev, theta_dev, C_tracks, gate, log_norm,
                       flags, row_ptr, col, val, ln_val, row_ptr_host, col_host, val_host, log_norm_host,
                       flags_host, stream=None, aux_stream=None, first_copy=None):
    """End-to-end step with C_k read back as the CSR of its gated entries (include/glmb.h).
    Host tensors pinned; returns nnz.  aux_stream (with prm.w_out set): reweight beside compat.
    first_copy: entries copied speculatively with row_ptr (default: the host capacity); more,
    up to the host capacity, in a second exact copy."""
    hp = lambda t: None if t is None else t.data_ptr()
    M = Z_host.shape[0]
    _check(load().glmb_step_host_csr(C.byref(prm), hp(Z_host), M, hp(theta_host), _ptr(Z_dev), _ptr(theta_dev),
                                     _ptr(C_tracks), C_tracks.shape[1], _ptr(gate), gate.shape[1], _ptr(log_norm),
                                     _ptr(flags), _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(ln_val), col.shape[0],
                                     hp(row_ptr_host), hp(col_host), hp(val_host), col_host.shape[0],
                                     col_host.shape[0] if first_copy is None else int(first_copy), hp(log_norm_host), hp(flags_host), _stream(stream),
                                     None if aux_stream is None else aux_stream.cuda_stream))
    return int(row_ptr_host[M])
