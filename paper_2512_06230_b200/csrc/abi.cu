// abi.cu -- the extern "C" boundary of libglmb.so (declared in include/glmb.h).
//
// Validation, device selection from the caller's stream, launch planning.
// Every entry point is asynchronous on the caller's stream (glmb_step_host
// excepted), never allocates, never aborts.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../include/glmb.h"
#include "glmb_internal.h"

namespace {

constexpr int kMaxDevices = 64;
int g_sm_count[kMaxDevices] = {0};
int g_checked[kMaxDevices] = {0};  // 0 unknown, 1 ok, -1 unsupported

glmb_status check_device(int dev) {
  if (dev < 0 || dev >= kMaxDevices) return GLMB_ERR_UNSUPPORTED_DEVICE;
  if (g_checked[dev] == 0) {
    int major = 0, minor = 0, sms = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      return GLMB_ERR_CUDA;
    }
    g_sm_count[dev] = sms;
    g_checked[dev] = (major == 10 && minor == 0) ? 1 : -1;
  }
  return g_checked[dev] == 1 ? GLMB_OK : GLMB_ERR_UNSUPPORTED_DEVICE;
}

// Make the stream's device current in this library's runtime instance.
glmb_status bind_stream(cudaStream_t s, int *dev_out) {
  int dev = 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (s != nullptr && cudaStreamIsCapturing(s, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone) {
    // inside a CUDA-graph capture: no stream queries (they would invalidate the capture);
    // the capturing thread's current device is the stream's
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      return GLMB_ERR_CUDA;
    }
    if (dev_out) *dev_out = dev;
    return check_device(dev);
  }
  if (s != nullptr) {
    if (cudaStreamGetDevice(s, &dev) != cudaSuccess) {
      cudaGetLastError();
      return GLMB_ERR_CUDA;
    }
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != dev) {
      if (cudaSetDevice(dev) != cudaSuccess) {
        cudaGetLastError();
        return GLMB_ERR_CUDA;
      }
    }
  } else if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return GLMB_ERR_CUDA;
  }
  if (dev_out) *dev_out = dev;
  return check_device(dev);
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

glmb_status check_particles(const glmb_particles *p, bool need_w, bool need_vpo) {
  if (p == nullptr) return GLMB_ERR_INVALID_ARG;
  if (p->n_tracks < 0) return GLMB_ERR_INVALID_ARG;
  if (p->n_tracks == 0) return GLMB_OK;
  if (p->n_particles < 4 || p->ld < p->n_particles) return GLMB_ERR_INVALID_ARG;
  if ((p->n_particles & 3) || (p->ld & 3)) return GLMB_ERR_ALIGNMENT;
  if (static_cast<int64_t>(p->n_tracks) * p->ld > (int64_t(1) << 40)) return GLMB_ERR_INVALID_ARG;
  const float *arr[6] = {p->x, p->y, p->v, p->psi, p->omega, p->w};
  const bool need[6] = {true, true, need_vpo, need_vpo, need_vpo, need_w};
  for (int k = 0; k < 6; ++k) {
    if (!need[k]) continue;
    if (arr[k] == nullptr) return GLMB_ERR_INVALID_ARG;
    if (!aligned16(arr[k])) return GLMB_ERR_ALIGNMENT;
  }
  return GLMB_OK;
}

bool spd(float Rxx, float Rxy, float Ryy) {
  const double det = static_cast<double>(Rxx) * Ryy - static_cast<double>(Rxy) * Rxy;
  return std::isfinite(det) && Rxx > 0.f && det > 0.0;
}

inline glmb_status from_cuda(cudaError_t e) { return e == cudaSuccess ? GLMB_OK : GLMB_ERR_CUDA; }

#define GLMB_TRY(expr)                    \
  do {                                    \
    const glmb_status st_ = (expr);       \
    if (st_ != GLMB_OK) return st_;       \
  } while (0)

// glmb_step_host with the C_k read-back overlapped: compat runs in track chunks
// (the same per-column arithmetic as one launch -- C is bit-identical under any
// split of the tracks), and each chunk's columns and gate words go back on
// copy_stream while the next chunk computes.
glmb_status step_host_overlapped(const glmb_step_params *prm, const float *Z_host, int32_t M,
                                 const int32_t *theta_host, float *Z_dev, int32_t *theta_dev, float *C_clutter_dev,
                                 float *C_tracks_dev, int64_t ldc, uint32_t *gate_dev, int64_t ldg,
                                 float *log_norm_dev, uint32_t *flags_dev, float *C_clutter_host,
                                 float *C_tracks_host, uint32_t *gate_host, float *log_norm_host,
                                 uint32_t *flags_host, cudaStream_t s, cudaStream_t cs);

}  // namespace

extern "C" {

int glmb_version(void) { return 10000; }

const char *glmb_status_string(glmb_status s) {
  switch (s) {
    case GLMB_OK: return "GLMB_OK";
    case GLMB_ERR_INVALID_ARG: return "GLMB_ERR_INVALID_ARG: argument violates the contract in glmb.h";
    case GLMB_ERR_ALIGNMENT: return "GLMB_ERR_ALIGNMENT: array not 16-B aligned or P/ld not a multiple of 4";
    case GLMB_ERR_UNSUPPORTED_DEVICE: return "GLMB_ERR_UNSUPPORTED_DEVICE: needs compute capability 10.0 (sm_100a)";
    case GLMB_ERR_CUDA: return "GLMB_ERR_CUDA: a CUDA call or kernel launch failed";
  }
  return "GLMB: unknown status";
}

glmb_status glmb_init(int device) {
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return GLMB_ERR_CUDA;
  }
  return check_device(device);
}

int glmb_sm_count(int device) {
  if (check_device(device) != GLMB_OK) return 0;
  return g_sm_count[device];
}

glmb_status glmb_predict(const glmb_particles *in, const glmb_particles *out, const int32_t *gid, float dt,
                         float sigma_a, float sigma_w, uint64_t seed, uint32_t step, glmb_stream_t stream) {
  GLMB_TRY(check_particles(in, false, true));
  GLMB_TRY(check_particles(out, false, true));
  if (in->n_tracks != out->n_tracks) return GLMB_ERR_INVALID_ARG;
  if (in->n_tracks > 0 && (in->n_particles != out->n_particles || in->ld != out->ld)) return GLMB_ERR_INVALID_ARG;
  if (!(dt > 0.f) || !(sigma_a >= 0.f) || !(sigma_w >= 0.f)) return GLMB_ERR_INVALID_ARG;
  if (in->n_tracks == 0) return GLMB_OK;
  if (gid == nullptr) return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  GLMB_TRY(bind_stream(s, &dev));
  glmb::PredictArgs a{in->x, in->y, in->v, in->psi, in->omega, out->x, out->y, out->v, out->psi, out->omega,
                      gid, in->n_tracks, in->n_particles, in->ld, dt, sigma_a, sigma_w,
                      static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), step};
  return from_cuda(glmb::launch_predict(a, g_sm_count[dev], s));
}

glmb_status glmb_birth(const glmb_particles *out, const int32_t *gid, const float *mean, const float *chol,
                       uint64_t seed, uint32_t step, glmb_stream_t stream) {
  GLMB_TRY(check_particles(out, true, true));
  if (out->n_tracks == 0) return GLMB_OK;
  if (gid == nullptr || mean == nullptr || chol == nullptr) return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  GLMB_TRY(bind_stream(s, &dev));
  glmb::BirthArgs a{out->x, out->y, out->v, out->psi, out->omega, out->w, gid, mean, chol,
                    out->n_tracks, out->n_particles, out->ld,
                    static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), step};
  return from_cuda(glmb::launch_birth(a, g_sm_count[dev], s));
}

namespace {
glmb_status compat_impl(const glmb_particles *trk, const float *Z, int32_t M, float Rxx, float Rxy, float Ryy,
                        float p_d, float kappa, float gamma, float *C_clutter, float *C_tracks, int64_t ldc,
                        uint32_t *gate, int64_t ldg, bool skip, unsigned long long *skipped, glmb_stream_t stream) {
  GLMB_TRY(check_particles(trk, true, false));
  if (M < 0) return GLMB_ERR_INVALID_ARG;
  if (!spd(Rxx, Rxy, Ryy) || !(p_d > 0.f && p_d <= 1.f) || !(kappa >= 0.f) || !(gamma >= 1e-30f))
    return GLMB_ERR_INVALID_ARG;
  if (M == 0) return GLMB_OK;
  if (Z == nullptr) return GLMB_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(Z) & 7u) != 0) return GLMB_ERR_ALIGNMENT;
  const int32_t T = trk->n_tracks;
  if (T > 0) {
    if (C_tracks == nullptr || gate == nullptr) return GLMB_ERR_INVALID_ARG;
    if (ldc < M || ldg < (M + 31) / 32) return GLMB_ERR_INVALID_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  if (T == 0) return from_cuda(glmb::launch_clutter_fill(C_clutter, M, kappa, s));

  // whitening: 1/2 log2(e) d^T R^-1 d = (a1 dx + a2 dy)^2 + (b2 dy)^2
  const double rxx = Rxx, rxy = Rxy, ryy = Ryy;
  const double det = rxx * ryy - rxy * rxy;
  const double s0 = std::sqrt(0.5 * 1.4426950408889634074);  // sqrt(1/2 log2 e)
  const double a1 = s0 * std::sqrt(ryy / det);
  const double a2 = -a1 * (rxy / ryy);
  const double b2 = s0 / std::sqrt(ryy);
  glmb::CompatArgs a{};
  a.x = trk->x; a.y = trk->y; a.w = trk->w; a.ld = trk->ld; a.T = T; a.P = trk->n_particles;
  a.Z = Z; a.M = M;
  a.a1 = static_cast<float>(a1); a.a2 = static_cast<float>(a2); a.b2 = static_cast<float>(b2);
  a.norm = static_cast<float>(1.0 / (2.0 * 3.14159265358979323846 * std::sqrt(det)));
  a.p_d = p_d; a.kappa = kappa; a.gamma = gamma;
  a.C_clutter = C_clutter; a.C_tracks = C_tracks; a.ldc = ldc; a.gate = gate; a.ldg = ldg;
  a.skip = skip ? 1 : 0;
  a.skip_count = skipped;
  glmb::compat_plan(M, a.P, &a.K, &a.NW, &a.CL, &a.n_mtiles);
  if (static_cast<int64_t>(T) * a.n_mtiles * a.CL > 0x7fffffffLL) return GLMB_ERR_INVALID_ARG;
  return from_cuda(glmb::launch_compat(a, s));
}
}  // namespace

glmb_status glmb_compat(const glmb_particles *trk, const float *Z, int32_t M, float Rxx, float Rxy, float Ryy,
                        float p_d, float kappa, float gamma, float *C_clutter, float *C_tracks, int64_t ldc,
                        uint32_t *gate, int64_t ldg, glmb_stream_t stream) {
  return compat_impl(trk, Z, M, Rxx, Rxy, Ryy, p_d, kappa, gamma, C_clutter, C_tracks, ldc, gate, ldg,
                     glmb::compat_skip_env(), nullptr, stream);
}

glmb_status glmb_compat_skipping(const glmb_particles *trk, const float *Z, int32_t M, float Rxx, float Rxy,
                                 float Ryy, float p_d, float kappa, float gamma, float *C_clutter, float *C_tracks,
                                 int64_t ldc, uint32_t *gate, int64_t ldg, uint64_t *skipped_pairs,
                                 glmb_stream_t stream) {
  return compat_impl(trk, Z, M, Rxx, Rxy, Ryy, p_d, kappa, gamma, C_clutter, C_tracks, ldc, gate, ldg, true,
                     reinterpret_cast<unsigned long long *>(skipped_pairs), stream);
}

glmb_status glmb_compat_peers(const glmb_particles *trk, const float *Z, int32_t M, float Rxx, float Rxy,
                              float Ryy, float p_d, float kappa, float gamma, float *C_clutter,
                              float *const *peer_C, uint32_t *const *peer_G, int32_t n_peers, int64_t row0,
                              int64_t ldc, int64_t ldg, glmb_stream_t stream) {
  GLMB_TRY(check_particles(trk, true, false));
  if (M < 0 || n_peers < 1 || n_peers > 64 || row0 < 0) return GLMB_ERR_INVALID_ARG;
  if (!spd(Rxx, Rxy, Ryy) || !(p_d > 0.f && p_d <= 1.f) || !(kappa >= 0.f) || !(gamma >= 1e-30f))
    return GLMB_ERR_INVALID_ARG;
  if (M == 0) return GLMB_OK;
  if (Z == nullptr || peer_C == nullptr || peer_G == nullptr) return GLMB_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(Z) & 7u) != 0) return GLMB_ERR_ALIGNMENT;
  if (ldc < M || ldg < (M + 31) / 32) return GLMB_ERR_INVALID_ARG;
  const int32_t T = trk->n_tracks;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  if (T == 0) return from_cuda(glmb::launch_clutter_fill(C_clutter, M, kappa, s));
  const double rxx = Rxx, rxy = Rxy, ryy = Ryy;
  const double det = rxx * ryy - rxy * rxy;
  const double s0 = std::sqrt(0.5 * 1.4426950408889634074);
  const double a1 = s0 * std::sqrt(ryy / det);
  glmb::CompatArgs a{};
  a.x = trk->x; a.y = trk->y; a.w = trk->w; a.ld = trk->ld; a.T = T; a.P = trk->n_particles;
  a.Z = Z; a.M = M;
  a.a1 = static_cast<float>(a1); a.a2 = static_cast<float>(-a1 * (rxy / ryy));
  a.b2 = static_cast<float>(s0 / std::sqrt(ryy));
  a.norm = static_cast<float>(1.0 / (2.0 * 3.14159265358979323846 * std::sqrt(det)));
  a.p_d = p_d; a.kappa = kappa; a.gamma = gamma;
  a.C_clutter = C_clutter; a.C_tracks = nullptr; a.ldc = ldc; a.gate = nullptr; a.ldg = ldg;
  a.peer_C = peer_C; a.peer_G = peer_G; a.n_peers = n_peers; a.peer_row0 = row0;
  a.skip = glmb::compat_skip_env() ? 1 : 0;
  glmb::compat_plan(M, a.P, &a.K, &a.NW, &a.CL, &a.n_mtiles);
  if (static_cast<int64_t>(T) * a.n_mtiles * a.CL > 0x7fffffffLL) return GLMB_ERR_INVALID_ARG;
  return from_cuda(glmb::launch_compat(a, s));
}

glmb_status glmb_reweight(const glmb_particles *trk, float *w_out, const float *Z, int32_t M, float Rxx, float Rxy,
                          float Ryy, const int32_t *theta, int32_t col_offset, float *log_norm, uint32_t *flags,
                          glmb_stream_t stream) {
  GLMB_TRY(check_particles(trk, true, false));
  if (trk->n_tracks > 0 && w_out == nullptr) return GLMB_ERR_INVALID_ARG;
  if (trk->n_tracks > 0 && (reinterpret_cast<uintptr_t>(w_out) & 15u) != 0) return GLMB_ERR_ALIGNMENT;
  if (M < 0 || !spd(Rxx, Rxy, Ryy)) return GLMB_ERR_INVALID_ARG;
  const int32_t T = trk->n_tracks;
  if (T == 0) return GLMB_OK;
  if (log_norm == nullptr || flags == nullptr) return GLMB_ERR_INVALID_ARG;
  if (M > 0 && (Z == nullptr || theta == nullptr)) return GLMB_ERR_INVALID_ARG;
  if (M > 0 && (reinterpret_cast<uintptr_t>(Z) & 7u) != 0) return GLMB_ERR_ALIGNMENT;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  const double rxx = Rxx, rxy = Rxy, ryy = Ryy;
  const double det = rxx * ryy - rxy * rxy;
  const double h = 0.5 * 1.4426950408889634074;  // 1/2 log2(e)
  glmb::ReweightArgs a{};
  a.x = trk->x; a.y = trk->y; a.w = trk->w; a.w_out = w_out; a.ld = trk->ld; a.T = T; a.P = trk->n_particles;
  a.Z = Z; a.M = M; a.theta = theta; a.col_offset = col_offset;
  a.qa = h * ryy / det;
  a.qb = -2.0 * h * rxy / det;
  a.qc = h * rxx / det;
  a.log_norm1 = std::log(2.0 * 3.14159265358979323846 * std::sqrt(det));
  a.log_norm = log_norm; a.flags = flags;
  a.ld_out = trk->ld;
  return from_cuda(glmb::launch_reweight(a, s));
}

glmb_status glmb_step(const glmb_step_params *prm, const float *Z, int32_t M, const int32_t *theta,
                      float *C_clutter, float *C_tracks, int64_t ldc, uint32_t *gate, int64_t ldg, float *log_norm,
                      uint32_t *flags, glmb_stream_t stream) {
  if (prm == nullptr) return GLMB_ERR_INVALID_ARG;
  const glmb_particles &all = prm->tracks;
  GLMB_TRY(check_particles(&all, true, true));
  const int32_t T = prm->n_survivors, Tk = all.n_tracks;
  if (T < 0 || T > Tk) return GLMB_ERR_INVALID_ARG;
  glmb_particles surv = all;
  surv.n_tracks = T;
  glmb_particles births = all;
  births.n_tracks = Tk - T;
  const int64_t off = static_cast<int64_t>(T) * all.ld;
  if (Tk > 0) {
    births.x = all.x + off; births.y = all.y + off; births.v = all.v + off;
    births.psi = all.psi + off; births.omega = all.omega + off; births.w = all.w + off;
  }
  GLMB_TRY(glmb_predict(&surv, &surv, prm->gid, prm->dt, prm->sigma_a, prm->sigma_w, prm->seed, prm->step, stream));
  GLMB_TRY(glmb_birth(&births, prm->gid ? prm->gid + T : nullptr, prm->birth_mean, prm->birth_chol, prm->seed,
                      prm->step, stream));
  GLMB_TRY(glmb_compat(&all, Z, M, prm->Rxx, prm->Rxy, prm->Ryy, prm->p_d, prm->kappa, prm->gamma, C_clutter,
                       C_tracks, ldc, gate, ldg, stream));
  return glmb_reweight(&all, prm->w_out ? prm->w_out : all.w, Z, M, prm->Rxx, prm->Rxy, prm->Ryy, theta,
                       prm->col_offset, log_norm, flags, stream);
}

glmb_status glmb_step_host(const glmb_step_params *prm, const float *Z_host, int32_t M, const int32_t *theta_host,
                           float *Z_dev, int32_t *theta_dev, float *C_clutter_dev, float *C_tracks_dev, int64_t ldc,
                           uint32_t *gate_dev, int64_t ldg, float *log_norm_dev, uint32_t *flags_dev,
                           float *C_clutter_host, float *C_tracks_host, uint32_t *gate_host, float *log_norm_host,
                           uint32_t *flags_host, glmb_stream_t stream, glmb_stream_t copy_stream) {
  if (prm == nullptr || M < 0) return GLMB_ERR_INVALID_ARG;
  if (copy_stream != nullptr && stream != nullptr)
    return step_host_overlapped(prm, Z_host, M, theta_host, Z_dev, theta_dev, C_clutter_dev, C_tracks_dev, ldc,
                                gate_dev, ldg, log_norm_dev, flags_dev, C_clutter_host, C_tracks_host, gate_host,
                                log_norm_host, flags_host, reinterpret_cast<cudaStream_t>(stream),
                                reinterpret_cast<cudaStream_t>(copy_stream));
  if (M > 0 && (Z_host == nullptr || theta_host == nullptr || Z_dev == nullptr || theta_dev == nullptr))
    return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  const int64_t Tk = prm->tracks.n_tracks;
  if (M > 0) {
    if (cudaMemcpyAsync(Z_dev, Z_host, sizeof(float) * 2 * M, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(theta_dev, theta_host, sizeof(int32_t) * M, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return GLMB_ERR_CUDA;
  }
  GLMB_TRY(glmb_step(prm, Z_dev, M, theta_dev, C_clutter_dev, C_tracks_dev, ldc, gate_dev, ldg, log_norm_dev,
                     flags_dev, stream));
  if (M > 0 && C_clutter_host && C_clutter_dev &&
      cudaMemcpyAsync(C_clutter_host, C_clutter_dev, sizeof(float) * M, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return GLMB_ERR_CUDA;
  if (Tk > 0 && M > 0) {
    if (C_tracks_host && cudaMemcpyAsync(C_tracks_host, C_tracks_dev, sizeof(float) * Tk * ldc,
                                         cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return GLMB_ERR_CUDA;
    if (gate_host && cudaMemcpyAsync(gate_host, gate_dev, sizeof(uint32_t) * Tk * ldg, cudaMemcpyDeviceToHost, s) !=
                         cudaSuccess)
      return GLMB_ERR_CUDA;
  }
  if (Tk > 0) {
    if (log_norm_host && cudaMemcpyAsync(log_norm_host, log_norm_dev, sizeof(float) * Tk, cudaMemcpyDeviceToHost,
                                         s) != cudaSuccess)
      return GLMB_ERR_CUDA;
    if (flags_host &&
        cudaMemcpyAsync(flags_host, flags_dev, sizeof(uint32_t) * Tk, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return GLMB_ERR_CUDA;
  }
  return from_cuda(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ hypothesis machinery
glmb_status glmb_death_prob(int32_t T, int32_t M, const float *C_tracks, int64_t ldc, const uint32_t *gate,
                            int64_t ldg, float p_d, float kappa, const float *p_s, float *d_out,
                            glmb_stream_t stream) {
  if (T < 0 || M < 0 || !(p_d > 0.f && p_d <= 1.f) || !(kappa >= 0.f)) return GLMB_ERR_INVALID_ARG;
  if (T == 0) return GLMB_OK;
  if (p_s == nullptr || d_out == nullptr) return GLMB_ERR_INVALID_ARG;
  if (M > 0 && (C_tracks == nullptr || gate == nullptr || ldc < M || ldg < (M + 31) / 32))
    return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  glmb::DeathArgs a{T, M, C_tracks, ldc, gate, ldg, p_d, kappa, p_s, d_out};
  return from_cuda(glmb::launch_death_prob(a, s));
}

glmb_status glmb_compat_rows(int32_t T, int32_t M, const float *C_tracks, int64_t ldc, const uint32_t *gate,
                             int64_t ldg, int32_t *row_ptr, int32_t *col, float *val, double *ln_val, int32_t cap,
                             glmb_stream_t stream) {
  if (T < 0 || M < 0 || cap < 0) return GLMB_ERR_INVALID_ARG;
  if (row_ptr == nullptr) return GLMB_ERR_INVALID_ARG;
  if (T > 0 && M > 0 && (C_tracks == nullptr || gate == nullptr || ldc < M || ldg < (M + 31) / 32))
    return GLMB_ERR_INVALID_ARG;
  if (cap > 0 && (col == nullptr || val == nullptr || ln_val == nullptr)) return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  GLMB_TRY(bind_stream(s, &dev));
  glmb::RowsArgs a{T, M, gate, ldg, C_tracks, ldc, row_ptr, col, val, ln_val, cap};
  return from_cuda(glmb::launch_compat_rows(a, g_sm_count[dev], s));
}

glmb_status glmb_assoc_sample(int32_t H_old, const int32_t *n_parents, int32_t H_up, int32_t T, int32_t M,
                              const uint32_t *parent_mask,
                              int32_t ldt, const double *parent_logw, const float *d_prob, const float *p_s,
                              float p_d, float kappa, const int32_t *row_ptr, const int32_t *col, const float *val,
                              const double *ln_val, const double *count_lp, int32_t n_count, uint64_t seed,
                              uint32_t step, uint32_t *alive, int32_t *theta, int64_t ldm, double *logw,
                              uint64_t *hash, glmb_stream_t stream) {
  if (H_old < 0 || H_up < 0 || T < 0 || M < 0) return GLMB_ERR_INVALID_ARG;
  if (H_up >= (1 << 24) || static_cast<int64_t>(H_old) * H_up > 0x7fffffffLL) return GLMB_ERR_INVALID_ARG;
  if (!(p_d > 0.f && p_d <= 1.f) || !(kappa >= 0.f)) return GLMB_ERR_INVALID_ARG;
  if (ldt < (T + 31) / 32 || ldt < 1 || ldt > 12 * 1024 || ldm < M) return GLMB_ERR_INVALID_ARG;
  if (n_count < 0 || (n_count > 0 && (count_lp == nullptr || T > 32768))) return GLMB_ERR_INVALID_ARG;
  if (static_cast<int64_t>(H_old) * H_up == 0) return GLMB_OK;
  if (parent_mask == nullptr || parent_logw == nullptr || alive == nullptr || logw == nullptr || row_ptr == nullptr)
    return GLMB_ERR_INVALID_ARG;
  if (T > 0 && (d_prob == nullptr || p_s == nullptr)) return GLMB_ERR_INVALID_ARG;
  if (M > 0 && (theta == nullptr || col == nullptr || val == nullptr || ln_val == nullptr))
    return GLMB_ERR_INVALID_ARG;
  if (M > 0 && ((ldm & 3) || (reinterpret_cast<uintptr_t>(theta) & 15u))) return GLMB_ERR_ALIGNMENT;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  GLMB_TRY(bind_stream(s, &dev));
  glmb::SampleArgs a{H_old, H_up, T, M, n_parents, parent_mask, ldt, parent_logw, d_prob, p_s, p_d, kappa, row_ptr, col, val,
                     ln_val, count_lp, n_count, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), step,
                     alive, theta, ldm,
                     logw, reinterpret_cast<unsigned long long *>(hash)};
  return from_cuda(glmb::launch_assoc_sample(a, g_sm_count[dev], s));
}

glmb_status glmb_dedup(int32_t H_old, const int32_t *n_parents, int32_t H_up, int32_t M, const uint32_t *alive,
                       int32_t ldt,
                       const int32_t *theta, int64_t ldm, const uint64_t *hash, uint8_t *unique,
                       glmb_stream_t stream) {
  if (H_old < 0 || H_up < 0 || M < 0 || ldt < 1 || ldm < M) return GLMB_ERR_INVALID_ARG;
  if (static_cast<int64_t>(H_old) * H_up == 0) return GLMB_OK;
  if (alive == nullptr || hash == nullptr || unique == nullptr || (M > 0 && theta == nullptr))
    return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  glmb::DedupArgs a{H_old, H_up, M, ldt, n_parents, ldm, alive, theta, reinterpret_cast<const unsigned long long *>(hash),
                    unique};
  return from_cuda(glmb::launch_dedup(a, s));
}

glmb_status glmb_prune(int32_t n, const double *logw, const uint8_t *unique, double tau, int32_t h_max,
                       uint64_t *workspace, int32_t *keep_idx, double *keep_w, int32_t *n_kept,
                       glmb_stream_t stream) {
  if (n < 0 || h_max < 0 || h_max > GLMB_PRUNE_HMAX_LIMIT || !(tau >= 0.0)) return GLMB_ERR_INVALID_ARG;
  if (n_kept == nullptr) return GLMB_ERR_INVALID_ARG;
  if (n > 0 && (logw == nullptr || unique == nullptr || workspace == nullptr)) return GLMB_ERR_INVALID_ARG;
  if (h_max > 0 && (keep_idx == nullptr || keep_w == nullptr)) return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  if (n == 0 || h_max == 0) return from_cuda(cudaMemsetAsync(n_kept, 0, sizeof(int32_t), s));
  glmb::PruneArgs a{n, logw, unique, tau, h_max, glmb::prune_capacity(h_max),
                    reinterpret_cast<unsigned long long *>(workspace), keep_idx, keep_w, n_kept};
  return from_cuda(glmb::launch_prune(a, s));
}

// ------------------------------------------------------------------ particle loop (f2)
size_t glmb_assoc_pairs_workspace_size(int32_t n_hyp, int32_t T, int32_t M) {
  if (n_hyp < 0 || T < 0 || M < 0) return 0;
  return glmb::pairs_workspace_bytes(n_hyp, T, M);
}

glmb_status glmb_assoc_pairs(int32_t n_hyp, const int32_t *n_hyp_dev, const int32_t *hyp_idx, const uint32_t *alive, int32_t ldt,
                             const int32_t *theta, int64_t ldm, int32_t T, int32_t M, int32_t *pair_track,
                             int32_t *pair_ptr, int32_t *pair_meas, int32_t *pair_of, int32_t *n_pairs,
                             void *workspace, size_t workspace_bytes, glmb_stream_t stream) {
  if (n_hyp < 0 || T < 0 || M < 0 || ldt < (T + 31) / 32 || ldt < 1 || ldm < M) return GLMB_ERR_INVALID_ARG;
  if (static_cast<int64_t>(n_hyp) * (T > M ? T : M) > 0x7fffffffLL) return GLMB_ERR_INVALID_ARG;
  if (static_cast<size_t>(T) * 12 > 200 * 1024) return GLMB_ERR_INVALID_ARG;  // per-track shared-memory tables
  if (n_pairs == nullptr || pair_ptr == nullptr) return GLMB_ERR_INVALID_ARG;
  if (n_hyp > 0 && T > 0) {
    if (hyp_idx == nullptr || alive == nullptr || pair_track == nullptr || pair_of == nullptr ||
        (M > 0 && (theta == nullptr || pair_meas == nullptr)))
      return GLMB_ERR_INVALID_ARG;
    if (workspace == nullptr || workspace_bytes < glmb::pairs_workspace_bytes(n_hyp, T, M))
      return GLMB_ERR_INVALID_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  glmb::PairsArgs a{};
  a.n_hyp = n_hyp; a.n_hyp_dev = n_hyp_dev; a.T = T; a.M = M; a.ldt = ldt; a.ldm = ldm; a.hyp_idx = hyp_idx; a.alive = alive;
  a.theta = theta; a.pair_track = pair_track; a.pair_ptr = pair_ptr; a.pair_meas = pair_meas;
  a.pair_of = pair_of; a.n_pairs = n_pairs;
  return from_cuda(glmb::launch_assoc_pairs(a, workspace, s));
}

glmb_status glmb_reweight_pairs(const glmb_particles *src, const float *Z, int32_t M, float Rxx, float Rxy,
                                float Ryy, int32_t K, const int32_t *n_pairs, const int32_t *pair_track,
                                const int32_t *pair_ptr, const int32_t *pair_meas, float *w_out, int64_t ld_out,
                                float *log_norm, uint32_t *flags, float *ess, glmb_stream_t stream) {
  GLMB_TRY(check_particles(src, true, false));
  if (K < 0 || M < 0 || !spd(Rxx, Rxy, Ryy)) return GLMB_ERR_INVALID_ARG;
  if (K == 0) return GLMB_OK;
  if (src->n_tracks == 0 || src->n_particles > GLMB_PAIRS_PMAX) return GLMB_ERR_INVALID_ARG;
  if (pair_track == nullptr || pair_ptr == nullptr || w_out == nullptr || log_norm == nullptr ||
      flags == nullptr || ess == nullptr)
    return GLMB_ERR_INVALID_ARG;
  if (M > 0 && (Z == nullptr || pair_meas == nullptr)) return GLMB_ERR_INVALID_ARG;
  if (ld_out < src->n_particles || (ld_out & 3)) return GLMB_ERR_ALIGNMENT;
  if ((reinterpret_cast<uintptr_t>(w_out) & 15u) != 0) return GLMB_ERR_ALIGNMENT;
  if (M > 0 && (reinterpret_cast<uintptr_t>(Z) & 7u) != 0) return GLMB_ERR_ALIGNMENT;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  GLMB_TRY(bind_stream(s, &dev));
  const double rxx = Rxx, rxy = Rxy, ryy = Ryy;
  const double det = rxx * ryy - rxy * rxy;
  const double h = 0.5 * 1.4426950408889634074;
  glmb::ReweightArgs a{};
  a.x = src->x; a.y = src->y; a.w = src->w; a.w_out = w_out; a.ld = src->ld; a.T = K; a.P = src->n_particles;
  a.Z = Z; a.M = M; a.theta = nullptr; a.col_offset = 0;
  a.qa = h * ryy / det;
  a.qb = -2.0 * h * rxy / det;
  a.qc = h * rxx / det;
  a.log_norm1 = std::log(2.0 * 3.14159265358979323846 * std::sqrt(det));
  a.log_norm = log_norm; a.flags = flags;
  a.pair_track = pair_track; a.pair_ptr = pair_ptr; a.pair_meas = pair_meas; a.n_units_dev = n_pairs;
  a.ld_out = ld_out; a.ess = ess;
  a.units_cap = 4 * (g_sm_count[dev] > 0 ? g_sm_count[dev] : 148);  // grid-stride over the device count
  return from_cuda(glmb::launch_reweight(a, s));
}

glmb_status glmb_resample(const glmb_particles *src, int32_t K, const int32_t *n_pairs, const int32_t *pair_track,
                          const float *w, int64_t ldw, const glmb_particles *out, uint64_t seed, uint32_t step,
                          uint32_t *flags, glmb_stream_t stream) {
  GLMB_TRY(check_particles(src, false, true));
  GLMB_TRY(check_particles(out, true, true));
  if (K < 0) return GLMB_ERR_INVALID_ARG;
  if (K == 0) return GLMB_OK;
  if (src->n_tracks == 0 || out->n_tracks < K || out->n_particles != src->n_particles ||
      src->n_particles > GLMB_PAIRS_PMAX)
    return GLMB_ERR_INVALID_ARG;
  if (pair_track == nullptr || w == nullptr) return GLMB_ERR_INVALID_ARG;
  if (ldw < src->n_particles || (ldw & 3) || (reinterpret_cast<uintptr_t>(w) & 15u)) return GLMB_ERR_ALIGNMENT;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  GLMB_TRY(bind_stream(s, &dev));
  glmb::ResampleArgs a{};
  a.x = src->x; a.y = src->y; a.v = src->v; a.psi = src->psi; a.omega = src->omega; a.ld = src->ld;
  a.P = src->n_particles; a.pair_track = pair_track; a.w = w; a.ldw = ldw; a.K = K; a.n_units_dev = n_pairs;
  a.ox = out->x; a.oy = out->y; a.ov = out->v; a.opsi = out->psi; a.oomega = out->omega; a.ow = out->w;
  a.ld_out = out->ld;
  a.key0 = static_cast<uint32_t>(seed); a.key1 = static_cast<uint32_t>(seed >> 32); a.step = step;
  a.flags = flags;
  return from_cuda(glmb::launch_resample(a, g_sm_count[dev], s));
}

// ------------------------------------------------------------------ tracker loop (f4)
glmb_status glmb_next_parents(int32_t n_hyp_cap, const int32_t *n_kept, const double *keep_w, const int32_t *pair_of,
                              int32_t T, int32_t K_cap, int32_t B, int32_t birth_col0, uint32_t *parent_mask,
                              int32_t ldt, double *parent_logw, int32_t *n_parents, const int32_t *birth_col0_dev,
                              glmb_stream_t stream) {
  if (n_hyp_cap < 0 || T < 0 || K_cap < 0 || B < 0 || birth_col0 < 0 || ldt < 1) return GLMB_ERR_INVALID_ARG;
  const int64_t col_max = birth_col0_dev != nullptr ? static_cast<int64_t>(K_cap) : static_cast<int64_t>(birth_col0);
  if (static_cast<int64_t>(K_cap) > 32LL * ldt || col_max + B > 32LL * ldt || ldt > 12 * 1024)
    return GLMB_ERR_INVALID_ARG;
  if (n_kept == nullptr || n_parents == nullptr) return GLMB_ERR_INVALID_ARG;
  if (n_hyp_cap > 0 && (keep_w == nullptr || parent_mask == nullptr || parent_logw == nullptr ||
                        (T > 0 && pair_of == nullptr)))
    return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  glmb::NextParentsArgs a{n_hyp_cap, n_kept, keep_w, pair_of, T, K_cap, B, birth_col0, ldt, parent_mask,
                          parent_logw, n_parents, birth_col0_dev};
  return from_cuda(glmb::launch_next_parents(a, s));
}

glmb_status glmb_map_estimate(const int32_t *n_kept, const int32_t *pair_of0, int32_t T, const glmb_particles *set,
                              double *est, glmb_stream_t stream) {
  if (T < 0 || n_kept == nullptr) return GLMB_ERR_INVALID_ARG;
  if (T == 0) return GLMB_OK;
  GLMB_TRY(check_particles(set, true, false));
  if (pair_of0 == nullptr || est == nullptr || set->n_tracks == 0) return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  glmb::MapEstimateArgs a{n_kept, pair_of0, T, set->n_particles, set->n_tracks, set->ld, set->x, set->y, set->w, est};
  return from_cuda(glmb::launch_map_estimate(a, s));
}

glmb_status glmb_update(const glmb_update_params *u, glmb_stream_t stream) {
  if (u == nullptr) return GLMB_ERR_INVALID_ARG;
  const int64_t n = static_cast<int64_t>(u->H_old) * u->H_up;
  {  // glmb_death_prob + glmb_compat_rows (same validation), the first two in one grid
    const int32_t T = u->T, M = u->M;
    if (T < 0 || M < 0 || u->rows_cap < 0 || u->row_ptr == nullptr) return GLMB_ERR_INVALID_ARG;
    if (!(u->p_d > 0.f && u->p_d <= 1.f) || !(u->kappa >= 0.f)) return GLMB_ERR_INVALID_ARG;
    if (T > 0 && (u->d_prob == nullptr || u->p_s == nullptr)) return GLMB_ERR_INVALID_ARG;
    if (T > 0 && M > 0 && (u->C_tracks == nullptr || u->gate == nullptr || u->ldc < M || u->ldg < (M + 31) / 32))
      return GLMB_ERR_INVALID_ARG;
    if (u->rows_cap > 0 && (u->col == nullptr || u->val == nullptr || u->ln_val == nullptr))
      return GLMB_ERR_INVALID_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int dev = 0;
    GLMB_TRY(bind_stream(s, &dev));
    glmb::DeathArgs d{T, M, u->C_tracks, u->ldc, u->gate, u->ldg, u->p_d, u->kappa, u->p_s, u->d_prob};
    glmb::RowsArgs r{T, M, u->gate, u->ldg, u->C_tracks, u->ldc, u->row_ptr, u->col, u->val, u->ln_val, u->rows_cap};
    GLMB_TRY(from_cuda(glmb::launch_death_and_rows(d, r, g_sm_count[dev], s)));
  }
  GLMB_TRY(glmb_assoc_sample(u->H_old, u->n_parents, u->H_up, u->T, u->M, u->parent_mask, u->ldt, u->parent_logw,
                             u->d_prob, u->p_s, u->p_d, u->kappa, u->row_ptr, u->col, u->val, u->ln_val, u->count_lp,
                             u->n_count, u->seed, u->step, u->alive, u->theta, u->ldm, u->logw, u->hash, stream));
  GLMB_TRY(glmb_dedup(u->H_old, u->n_parents, u->H_up, u->M, u->alive, u->ldt, u->theta, u->ldm, u->hash, u->unique,
                      stream));
  if (n > 0x7fffffffLL) return GLMB_ERR_INVALID_ARG;
  GLMB_TRY(glmb_prune(static_cast<int32_t>(n), u->logw, u->unique, u->tau, u->h_max, u->prune_ws, u->keep_idx,
                      u->keep_w, u->n_kept, stream));
  GLMB_TRY(glmb_assoc_pairs(u->h_max, u->n_kept, u->keep_idx, u->alive, u->ldt, u->theta, u->ldm, u->T, u->M,
                            u->pair_track, u->pair_ptr, u->pair_meas, u->pair_of, u->n_pairs, u->pairs_ws,
                            u->pairs_ws_bytes, stream));
  const int32_t K = static_cast<int32_t>(std::min<int64_t>(u->K_cap, std::max<int64_t>(1, static_cast<int64_t>(u->h_max) * u->T)));
  GLMB_TRY(glmb_reweight_pairs(&u->tracks, u->Z, u->M, u->Rxx, u->Rxy, u->Ryy, K, u->n_pairs, u->pair_track,
                               u->pair_ptr, u->pair_meas, u->w_new, u->ld_new, u->log_norm, u->flags, u->ess, stream));
  GLMB_TRY(glmb_resample(&u->tracks, K, u->n_pairs, u->pair_track, u->w_new, u->ld_new, &u->out, u->seed, u->step,
                         u->flags, stream));
  if (u->est != nullptr) GLMB_TRY(glmb_map_estimate(u->n_kept, u->pair_of, u->T, &u->out, u->est, stream));
  return GLMB_OK;
}

glmb_status glmb_step_host_csr(const glmb_step_params *prm, const float *Z_host, int32_t M,
                               const int32_t *theta_host, float *Z_dev, int32_t *theta_dev, float *C_tracks_dev,
                               int64_t ldc, uint32_t *gate_dev, int64_t ldg, float *log_norm_dev, uint32_t *flags_dev,
                               int32_t *row_ptr_dev, int32_t *col_dev, float *val_dev, double *ln_val_dev,
                               int32_t cap, int32_t *row_ptr_host, int32_t *col_host, float *val_host,
                               int32_t cap_host, int32_t first_host, float *log_norm_host, uint32_t *flags_host,
                               glmb_stream_t stream, glmb_stream_t aux_stream) {
  if (prm == nullptr || M < 0 || cap < 0 || cap_host < 0 || first_host < 0) return GLMB_ERR_INVALID_ARG;
  if (M > 0 && (Z_host == nullptr || theta_host == nullptr || Z_dev == nullptr || theta_dev == nullptr))
    return GLMB_ERR_INVALID_ARG;
  if (row_ptr_dev == nullptr || row_ptr_host == nullptr) return GLMB_ERR_INVALID_ARG;
  if (cap_host > 0 && (col_host == nullptr || val_host == nullptr)) return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  const int32_t Tk = prm->tracks.n_tracks;
  if (M > 0) {
    if (cudaMemcpyAsync(Z_dev, Z_host, sizeof(float) * 2 * M, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(theta_dev, theta_host, sizeof(int32_t) * M, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return GLMB_ERR_CUDA;
  }
  // out of place with an aux stream: reweight (reads w, writes prm->w_out) runs on aux_stream
  // beside compat, enqueued first (a kernel queued behind compat only gets SMs in its tail)
  const bool overlap = prm->w_out != nullptr && aux_stream != nullptr && stream != nullptr;
  cudaStream_t as = reinterpret_cast<cudaStream_t>(aux_stream);
  cudaEvent_t ev = nullptr;
  if (!overlap) {
    GLMB_TRY(glmb_step(prm, Z_dev, M, theta_dev, nullptr, C_tracks_dev, ldc, gate_dev, ldg, log_norm_dev, flags_dev,
                       stream));
  } else {
    const glmb_particles &all = prm->tracks;
    GLMB_TRY(check_particles(&all, true, true));
    const int32_t T = prm->n_survivors;
    if (T < 0 || T > Tk) return GLMB_ERR_INVALID_ARG;
    glmb_particles surv = all, births = all;
    surv.n_tracks = T;
    births.n_tracks = Tk - T;
    const int64_t off = static_cast<int64_t>(T) * all.ld;
    if (Tk > 0) {
      births.x = all.x + off; births.y = all.y + off; births.v = all.v + off;
      births.psi = all.psi + off; births.omega = all.omega + off; births.w = all.w + off;
    }
    GLMB_TRY(glmb_predict(&surv, &surv, prm->gid, prm->dt, prm->sigma_a, prm->sigma_w, prm->seed, prm->step, stream));
    GLMB_TRY(glmb_birth(&births, prm->gid ? prm->gid + T : nullptr, prm->birth_mean, prm->birth_chol, prm->seed,
                        prm->step, stream));
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return GLMB_ERR_CUDA;
    glmb_status st = GLMB_OK;
    if (cudaEventRecord(ev, s) != cudaSuccess || cudaStreamWaitEvent(as, ev, 0) != cudaSuccess) st = GLMB_ERR_CUDA;
    if (st == GLMB_OK)
      st = glmb_reweight(&all, prm->w_out, Z_dev, M, prm->Rxx, prm->Rxy, prm->Ryy, theta_dev, prm->col_offset,
                         log_norm_dev, flags_dev, aux_stream);
    if (st == GLMB_OK)
      st = glmb_compat(&all, Z_dev, M, prm->Rxx, prm->Rxy, prm->Ryy, prm->p_d, prm->kappa, prm->gamma, nullptr,
                       C_tracks_dev, ldc, gate_dev, ldg, stream);
    cudaEventDestroy(ev);
    if (st != GLMB_OK) return st;
  }
  GLMB_TRY(glmb_compat_rows(Tk, M, C_tracks_dev, ldc, gate_dev, ldg, row_ptr_dev, col_dev, val_dev, ln_val_dev, cap,
                            stream));
  // one read-back: row_ptr, the first first_host entries (speculative), log_norm, flags; the
  // rest only if the gated entries outnumber them (then a second, exact-size copy, up to cap_host)
  const int32_t first = std::min(std::min(first_host, cap_host), cap);
  if (cudaMemcpyAsync(row_ptr_host, row_ptr_dev, sizeof(int32_t) * (M + 1), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return GLMB_ERR_CUDA;
  if (first > 0 &&
      (cudaMemcpyAsync(col_host, col_dev, sizeof(int32_t) * first, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
       cudaMemcpyAsync(val_host, val_dev, sizeof(float) * first, cudaMemcpyDeviceToHost, s) != cudaSuccess))
    return GLMB_ERR_CUDA;
  if (Tk > 0) {
    cudaStream_t ls = overlap ? as : s;  // log_norm / flags from reweight's stream
    if (log_norm_host && cudaMemcpyAsync(log_norm_host, log_norm_dev, sizeof(float) * Tk, cudaMemcpyDeviceToHost,
                                         ls) != cudaSuccess)
      return GLMB_ERR_CUDA;
    if (flags_host &&
        cudaMemcpyAsync(flags_host, flags_dev, sizeof(uint32_t) * Tk, cudaMemcpyDeviceToHost, ls) != cudaSuccess)
      return GLMB_ERR_CUDA;
  }
  if (cudaStreamSynchronize(s) != cudaSuccess) return GLMB_ERR_CUDA;
  if (overlap && cudaStreamSynchronize(as) != cudaSuccess) return GLMB_ERR_CUDA;
  const int32_t nnz = row_ptr_host[M];
  if (nnz > cap) return GLMB_ERR_INVALID_ARG;  /* device CSR capacity too small: entries past cap lost */
  if (nnz > first) {
    if (nnz > cap_host) return GLMB_ERR_INVALID_ARG;
    if (cudaMemcpyAsync(col_host + first, col_dev + first, sizeof(int32_t) * (nnz - first), cudaMemcpyDeviceToHost,
                        s) != cudaSuccess ||
        cudaMemcpyAsync(val_host + first, val_dev + first, sizeof(float) * (nnz - first), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess)
      return GLMB_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return GLMB_ERR_CUDA;
  }
  return GLMB_OK;
}

glmb_status glmb_philox_dump(uint64_t seed, const uint32_t *ctr, int32_t N, uint32_t *out, glmb_stream_t stream) {
  if (N < 0 || (N > 0 && (ctr == nullptr || out == nullptr))) return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  return from_cuda(glmb::launch_philox_dump(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), ctr, N,
                                            out, s));
}

glmb_status glmb_normals_dump(uint64_t seed, const uint32_t *ctr, int32_t N, float *out, glmb_stream_t stream) {
  if (N < 0 || (N > 0 && (ctr == nullptr || out == nullptr))) return GLMB_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  GLMB_TRY(bind_stream(s, nullptr));
  return from_cuda(glmb::launch_normals_dump(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), ctr, N,
                                             out, s));
}

}  // extern "C"

namespace {

glmb_status step_host_overlapped(const glmb_step_params *prm, const float *Z_host, int32_t M,
                                 const int32_t *theta_host, float *Z_dev, int32_t *theta_dev, float *C_clutter_dev,
                                 float *C_tracks_dev, int64_t ldc, uint32_t *gate_dev, int64_t ldg,
                                 float *log_norm_dev, uint32_t *flags_dev, float *C_clutter_host,
                                 float *C_tracks_host, uint32_t *gate_host, float *log_norm_host,
                                 uint32_t *flags_host, cudaStream_t s, cudaStream_t cs) {
  const glmb_particles &all = prm->tracks;
  GLMB_TRY(check_particles(&all, true, true));
  const int32_t T = prm->n_survivors, Tk = all.n_tracks;
  if (T < 0 || T > Tk) return GLMB_ERR_INVALID_ARG;
  if (M > 0 && (Z_host == nullptr || theta_host == nullptr || Z_dev == nullptr || theta_dev == nullptr))
    return GLMB_ERR_INVALID_ARG;
  GLMB_TRY(bind_stream(s, nullptr));
  if (M > 0) {
    if (cudaMemcpyAsync(Z_dev, Z_host, sizeof(float) * 2 * M, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(theta_dev, theta_host, sizeof(int32_t) * M, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return GLMB_ERR_CUDA;
  }
  auto rows = [&](int32_t r0, int32_t r1) {
    glmb_particles v = all;
    v.n_tracks = r1 - r0;
    const int64_t off = static_cast<int64_t>(r0) * all.ld;
    if (Tk > 0) {
      v.x = all.x + off; v.y = all.y + off; v.v = all.v + off;
      v.psi = all.psi + off; v.omega = all.omega + off; v.w = all.w + off;
    }
    return v;
  };
  glmb_particles surv = rows(0, T), births = rows(T, Tk);
  glmb_stream_t st = reinterpret_cast<glmb_stream_t>(s);
  GLMB_TRY(glmb_predict(&surv, &surv, prm->gid, prm->dt, prm->sigma_a, prm->sigma_w, prm->seed, prm->step, st));
  GLMB_TRY(glmb_birth(&births, prm->gid ? prm->gid + T : nullptr, prm->birth_mean, prm->birth_chol, prm->seed,
                      prm->step, st));
  // compat chunks: GLMB_HOST_CHUNKS (1..4, default 1: one launch, its read-back overlapping
  // reweight; more chunks overlap the read-back with compat too but pay a partial wave each)
  static const int chunks_env = [] {
    const char *e = std::getenv("GLMB_HOST_CHUNKS");
    const int v = e ? std::atoi(e) : 1;
    return v >= 1 && v <= 4 ? v : 1;
  }();
  constexpr int kMaxChunks = 4;
  const int kChunks = chunks_env;
  cudaEvent_t ev[kMaxChunks] = {};
  glmb_status status = GLMB_OK;
  // compat (chunks) on `s`, then reweight on `s` (into prm->w_out when given); the copy
  // stream reads each compat chunk's columns back while the next chunk / reweight runs.
  // (Reweight on the copy stream concurrently with compat was measured slower: compat
  // holds every SM, so reweight ran after it and delayed the read-back queued behind it.)
  struct Chunk {
    int32_t r0, r1;
  } chunk[kMaxChunks];
  int n_chunk = 0;
  const int32_t per = (Tk + kChunks - 1) / kChunks;
  for (int c = 0; c < kChunks && status == GLMB_OK; ++c) {
    const int32_t r0 = std::min(Tk, c * per), r1 = std::min(Tk, r0 + per);
    if (r1 <= r0 && c > 0) break;
    glmb_particles v = rows(r0, r1);
    status = glmb_compat(&v, Z_dev, M, prm->Rxx, prm->Rxy, prm->Ryy, prm->p_d, prm->kappa, prm->gamma,
                         c == 0 ? C_clutter_dev : nullptr, C_tracks_dev + static_cast<int64_t>(r0) * ldc, ldc,
                         gate_dev + static_cast<int64_t>(r0) * ldg, ldg, st);
    if (status != GLMB_OK || M == 0 || r1 <= r0) continue;
    if (cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev[c], s) != cudaSuccess) {
      status = GLMB_ERR_CUDA;
      break;
    }
    chunk[n_chunk++] = Chunk{r0, r1};
  }
  for (int c = 0; c < n_chunk && status == GLMB_OK; ++c) {
    const int32_t r0 = chunk[c].r0, r1 = chunk[c].r1;
    if (cudaStreamWaitEvent(cs, ev[c], 0) != cudaSuccess) {
      status = GLMB_ERR_CUDA;
      break;
    }
    if (C_tracks_host &&
        cudaMemcpyAsync(C_tracks_host + static_cast<int64_t>(r0) * ldc, C_tracks_dev + static_cast<int64_t>(r0) * ldc,
                        sizeof(float) * (r1 - r0) * ldc, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
      status = GLMB_ERR_CUDA;
    if (gate_host &&
        cudaMemcpyAsync(gate_host + static_cast<int64_t>(r0) * ldg, gate_dev + static_cast<int64_t>(r0) * ldg,
                        sizeof(uint32_t) * (r1 - r0) * ldg, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
      status = GLMB_ERR_CUDA;
  }
  if (status == GLMB_OK)
    status = glmb_reweight(&all, prm->w_out ? prm->w_out : all.w, Z_dev, M, prm->Rxx, prm->Rxy, prm->Ryy, theta_dev,
                           prm->col_offset, log_norm_dev, flags_dev, st);
  if (status == GLMB_OK) {
    cudaStream_t ls = s;
    if (M > 0 && C_clutter_host && C_clutter_dev &&
        cudaMemcpyAsync(C_clutter_host, C_clutter_dev, sizeof(float) * M, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      status = GLMB_ERR_CUDA;
    if (Tk > 0 && log_norm_host &&
        cudaMemcpyAsync(log_norm_host, log_norm_dev, sizeof(float) * Tk, cudaMemcpyDeviceToHost, ls) != cudaSuccess)
      status = GLMB_ERR_CUDA;
    if (Tk > 0 && flags_host &&
        cudaMemcpyAsync(flags_host, flags_dev, sizeof(uint32_t) * Tk, cudaMemcpyDeviceToHost, ls) != cudaSuccess)
      status = GLMB_ERR_CUDA;
  }
  const bool ok_sync = cudaStreamSynchronize(s) == cudaSuccess && cudaStreamSynchronize(cs) == cudaSuccess;
  for (int c = 0; c < kMaxChunks; ++c)
    if (ev[c]) cudaEventDestroy(ev[c]);
  if (status == GLMB_OK && !ok_sync) status = GLMB_ERR_CUDA;
  return status;
}

}  // namespace
