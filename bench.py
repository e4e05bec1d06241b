#!/usr/bin/env python
"""bench.py -- one GLMB step core (predict + birth + compat + reweight) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl glmb|reference]

Metric (BASELINE.json): particle-measurement likelihood evals/s (whole job,
all ranks) and ms per GLMB step.  Evals per step = M_k*T_k*P (compat, the
dense mixture) + P*#{i: theta_i != 0} (reweight).  Workload: BASELINE config 3
(T=1024+16 births, P=8192, M~1200) at N=1; config 4 (T=4096, P=8192, M~4800,
tracks sharded, Z/theta broadcast, C all-gathered over NCCL) at N>1.

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
synchronize, CUDA events on the launching stream, max over ranks.  Inputs
(particle state 204 MB at cfg3, > 126 MB L2) stream through HBM every step.
Rank 0 prints one JSON line.  The oracle (oracle/, fp64 CPU) is executed only
in the cpu_baseline leg and in --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-measurement likelihood evals/s (GLMB step: predict+birth+compat+reweight)"
# measured on B200 by glmb_peaks (profiles/r01_peaks.json, at the 1965 MHz max clock):
SFU_EX2_PER_CLK_PER_SM = 15.94       # MUFU.EX2 results/clk/SM (nominal 16)
FMA_LANES_PER_CLK_PER_SM = 124.0     # FP32 lanes/clk/SM issued as FFMA2 (nominal 128; plain FFMA 120.4)
# compat, per pair (exact-difference form): 5 FP32 lane-ops (dx, dy, dx^2, +dy^2, acc) + one exp;
# an exp moved to the FMA pipe costs 8 FP32 lane-ops.
# Best split f of exps on the FMA pipe: x(1-f) = E, x(5+8f) = F  ->  x = (F + 8E) / 13 pairs/clk/SM.
COMPAT_PAIRS_PER_CLK_PER_SM = (FMA_LANES_PER_CLK_PER_SM + 8 * SFU_EX2_PER_CLK_PER_SM) / 13.0
HBM_PEAK_GBPS_FALLBACK = 6556.5      # MEASURED_PEAKS.json hbm_gbs (read at run time when present)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=None)
    ap.add_argument("--impl", default="glmb", choices=["glmb", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--no-update", action="store_true", help="skip the GLMB update (f1-f3) timing")
    ap.add_argument("--h-old", type=int, default=100)
    ap.add_argument("--h-up", type=int, default=100)
    ap.add_argument("--h-max", type=int, default=100)
    ap.add_argument("--no-convoy", action="store_true", help="skip the paper-shaped convoy run (f4)")
    ap.add_argument("--no-graphs", action="store_true", help="skip the CUDA-graph timing of configs 0-2")
    ap.add_argument("--no-skip-probe", action="store_true", help="skip the exact zero-tile skipping probe")
    ap.add_argument("--no-b2b", action="store_true",
                    help="skip the back-to-back launch timing of the HBM-bound kernels (ncu launch lists)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Polls NVML every 2 ms while active: SM clock, max clock, throttle reasons."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            # the main thread spends the timed region enqueueing steps from Python: a short
            # GIL switch interval lets the poller run every few ms (one sample otherwise)
            self._switch = sys.getswitchinterval()
            sys.setswitchinterval(0.0005)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            sys.setswitchinterval(self._switch)

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "samples": len(self.samples), "reasons": sorted(self.reasons)}


# ------------------------------------------------------------------ CPU oracle legs
class OracleSample:
    """The fp64 oracle (as it stands) on a bounded sample of the workload: the
    first n tracks of the config -- predict, compat over all M, reweight -- with
    OpenMP over tracks.  n is calibrated once so one run takes ~`seconds`."""

    def __init__(self, cfg_id: int, seconds: float, cores: int):
        import oracle
        from paper_2512_06230_b200.scenes import make_scene
        self.oracle, self.make_scene = oracle, make_scene
        oracle.set_num_threads(cores)
        self.cfg_id, self.cores = cfg_id, cores
        base = make_scene(cfg_id, rows=range(0), steps=1)
        self.c = base.cfg
        self.Z, self.th = base.Z[0], base.theta[0]
        n0 = max(1, min(self.c.T, cores))
        t0, _ = self.run(n0)
        n = int(min(self.c.T, max(n0, n0 * seconds / max(t0, 1e-3))))
        self.n = max(n0, (n // n0) * n0)

    def run(self, n: int = None):
        n = self.n if n is None else n
        c, o = self.c, self.oracle
        s = self.make_scene(self.cfg_id, rows=range(n), steps=1)
        t0 = time.perf_counter()
        px, py, _, _, _ = o.predict(s.x, s.y, s.v, s.psi, s.omega, s.gid, c.dt, c.sigma_a,
                                    c.sigma_w, c.seed, 0)
        x32, y32 = px.astype(np.float32), py.astype(np.float32)
        o.compat(x32, y32, s.w, self.Z, c.R, c.p_d, c.kappa, c.gamma)
        o.reweight(x32, y32, s.w, self.Z, c.R, self.th, 0)
        dt = time.perf_counter() - t0
        n_assigned = int(((self.th >= 1) & (self.th <= n)).sum())
        return dt, len(self.Z) * n * c.P + c.P * n_assigned

    def describe(self, dt):
        c = self.c
        return (f"cfg{self.cfg_id}: first {self.n} of {c.T + c.B} tracks x all M={len(self.Z)} x "
                f"P={c.P} (predict+compat+reweight, fp64, OpenMP over tracks), {dt:.2f} s")


def oracle_sample(cfg_id: int, seconds: float, cores: int, single_core: bool = True):
    """The oracle on all `cores` host threads (the reported baseline) and, beside it, on one
    thread with a third of the time budget (oracle at 1 and all host cores)."""
    smp = OracleSample(cfg_id, seconds, cores)
    dt, evals = smp.run()
    out = {"value": evals / dt, "unit": "evals/s", "cores": cores, "kind": "oracle",
           "sample": smp.describe(dt)}
    if single_core and cores > 1:
        one = OracleSample(cfg_id, seconds / 3, 1)
        dt1, ev1 = one.run()
        out["single_core"] = {"value": ev1 / dt1, "unit": "evals/s", "cores": 1, "sample": one.describe(dt1)}
    return out


def workload_config(cfg_id, cfg, world, M_mean, evals_per_step):
    """The `config` object both arms print (same keys and values for the same workload)."""
    return {"workload": f"cfg{cfg_id} ({cfg.name})", "T": cfg.T, "B": cfg.B, "P": cfg.P, "M_mean": M_mean,
            "parallelism": f"tracks sharded x{world}",
            "l2": f"inputs larger than L2: particle state 24 B x T_k x P "
                  f"({24 * (cfg.T + cfg.B) * cfg.P / 1e6:.0f} MB) streams from HBM every step",
            "evals_per_step": evals_per_step}


class OracleStep:
    """The fp64 oracle running the bench's workload step by step (the reference arm): predict
    of the survivors (O5), births (O6), compat over [survivors | births] x all M_k (O7),
    reweight under theta_k (O8), the state (fp32-rounded, as the GPU keeps it) carried from
    step to step -- the same steps, step indices and measurements the GPU arm times.  n_tracks
    < T samples the first n survivor tracks (and all births) when the whole step would not fit
    the time budget; at config 3 on the box's 16 cores the whole step fits (~6 s)."""

    def __init__(self, cfg_id: int, n_steps: int, n_tracks: int, cores: int):
        import oracle
        from paper_2512_06230_b200.scenes import make_scene
        self.o = oracle
        oracle.set_num_threads(cores)
        self.cfg_id, self.cores = cfg_id, cores
        s = make_scene(cfg_id, rows=range(n_tracks), steps=n_steps)
        self.s, self.c, self.n = s, s.cfg, n_tracks
        self.state = [a.astype(np.float32) for a in (s.x, s.y, s.v, s.psi, s.omega, s.w)]

    def step(self, k: int):
        s, c, o = self.s, self.c, self.o
        zi = k % len(s.Z)
        Z, th = s.Z[zi], s.theta[zi]
        t0 = time.perf_counter()
        x, y, v, psi, om, w = self.state
        pred = [a.astype(np.float32) for a in o.predict(x, y, v, psi, om, s.gid, c.dt, c.sigma_a, c.sigma_w,
                                                         c.seed, k)]
        if c.B:
            b = [a.astype(np.float32) for a in o.birth(s.birth_mean, s.birth_chol, s.birth_gid, c.P, c.seed, k)]
            cols = [np.concatenate([pa, ba]) for pa, ba in zip(pred + [w], b)]
        else:
            cols = pred + [w]
        o.compat(cols[0], cols[1], cols[5], Z, c.R, c.p_d, c.kappa, c.gamma)
        # theta's columns are global: the sampled survivors keep theirs, births sit at T + b
        th_s = np.where((th >= 1) & (th <= self.n), th,
                        np.where(th > c.T, th - (c.T - self.n), 0)).astype(np.int32)
        w_new = o.reweight(cols[0], cols[1], cols[5], Z, c.R, th_s, 0)[0].astype(np.float32)
        dt = time.perf_counter() - t0
        self.state = pred + [w_new[:self.n]]
        n_cols = self.n + c.B
        n_assigned = int((th_s != 0).sum())
        return dt, len(Z) * n_cols * c.P + c.P * n_assigned

    def describe(self):
        c = self.c
        what = "every track" if self.n == c.T else f"the first {self.n} of {c.T} survivor tracks + all {c.B} births"
        return (f"cfg{self.cfg_id}: {what} x all M_k x P={c.P}; predict + birth + compat + reweight per step, "
                f"state carried, fp64, OpenMP over tracks on {self.cores} threads")


def reference_arm(a, cfg_id, budget_s: float = 240.0):
    """--impl reference: this tier's reference is the fp64 oracle (there is no reference
    implementation, only the paper), timed as it stands on the host's cores over the same
    workload steps as the GPU arm.  The whole step is run when K + W steps fit `budget_s`
    (config 3), else the first n survivor tracks (config 4 at N > 1).  Rank 0 alone runs it;
    the other ranks exit 0."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2512_06230_b200.scenes import CONFIGS
    cfg = CONFIGS[cfg_id]
    cores = host_cores()
    n_steps = max(cfg.steps, a.warmup + a.steps)   # the GPU arm's steps use the same Z_k (prefix-stable)
    # calibrate on a few tracks: seconds per track-step
    n0 = max(1, min(cfg.T, cores))
    cal = OracleStep(cfg_id, n_steps, n0, cores)
    t_cal, _ = cal.step(0)
    per_track = t_cal / (n0 + cfg.B)
    per_step_budget = budget_s / max(1, a.steps + a.warmup)
    n = cfg.T if per_track * (cfg.T + cfg.B) <= per_step_budget else \
        max(n0, min(cfg.T, int(per_step_budget / per_track) - cfg.B))
    smp = OracleStep(cfg_id, n_steps, n, cores)
    times, evals, Ms, full_ev = [], [], [], []
    for k in range(a.warmup + a.steps):
        dt, ev = smp.step(k)
        if k >= a.warmup:
            times.append(dt)
            evals.append(ev)
            zi = k % len(smp.s.Z)
            Ms.append(len(smp.s.Z[zi]))
            full_ev.append(len(smp.s.Z[zi]) * (cfg.T + cfg.B) * cfg.P + cfg.P * int((smp.s.theta[zi] != 0).sum()))
    value = sum(evals) / sum(times)
    M_mean = float(np.mean(Ms))
    full_evals = M_mean * (cfg.T + cfg.B) * cfg.P
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg_id, cfg, world, M_mean, float(sum(full_ev)) / a.steps),
            "sample": smp.describe() + ("" if n == cfg.T else
                                        f"; ms_per_step is the sampled step's (the whole step would be "
                                        f"~{1e3 * full_evals / value:.0f} ms at this rate)"),
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "oracle",
                             "sample": smp.describe()},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def hbm_peak() -> float:
    """MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth), else the fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return HBM_PEAK_GBPS_FALLBACK


def compat_traffic(T: int, P: int, M: int):
    """DRAM bytes per compat launch for this workload from the committed
    ncu --set full capture (profiles/compat_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "compat_traffic.json")) as f:
            return json.load(f).get(f"T{T}_P{P}_M{M}")
    except Exception:  # noqa: BLE001
        return None


def reweight_bytes(st, k: int) -> int:
    """Algorithmic bytes of step k's reweight on this rank: x, y, w read and w written (16 B per
    particle) for a track with an assigned measurement, w copied (8 B) for one without."""
    th = np.asarray(st.scene.theta[k % len(st.scene.theta)])
    cols = set(int(c) - 1 for c in th[th > 0])
    hit = sum(1 for c in st.col_of_row if int(c) in cols)
    return st.P * (16 * hit + 8 * (st.T_local - hit))


def hbm_back_to_back(st, stream, dev, k: int):
    """Back-to-back launch durations of the step's HBM-bound kernels on the current state:
    predict (survivors into a scratch state) and reweight (new weights into a scratch
    buffer) -- every launch reads the same inputs and writes the same scratch, so the
    state of the timed steps is untouched."""
    import torch
    from paper_2512_06230_b200 import _lib as L
    out = {}
    scratch = L.Particles(torch.empty_like(st.particles.data), st.P)
    if st.T_surv:
        src, dst = st.survivors(), scratch.rows(0, st.T_surv)
        out["predict"] = back_to_back_ms(
            lambda: L.glmb_predict(src, dst, st.gid[:st.T_surv], st.cfg.dt, st.cfg.sigma_a, st.cfg.sigma_w,
                                   st.seed, k, stream), stream, dev)
    if st.contiguous and st.T_local:
        zi = k % len(st.Z)
        w_out = torch.empty_like(st.weights())
        ln, fl = torch.empty_like(st.out.log_norm), torch.empty_like(st.out.flags)
        out["reweight"] = back_to_back_ms(
            lambda: L.glmb_reweight(st.particles, st.Z[zi], st.R, st.theta[zi], st.col_offset, ln, fl, stream,
                                    w_out=w_out), stream, dev)
    del scratch
    return out


def back_to_back_ms(fn, stream, dev, reps: int = 10, trials: int = 5) -> float:
    """Mean launch duration of `fn` (one kernel launch on `stream`) over `reps` launches back to
    back between two events, queued behind a busy GPU so no host gap enters; median of
    `trials`.  A single launch between two events also carries a fixed ~8 us of event and
    launch overhead (profiles/reweight_time.py), which this amortises."""
    import torch
    out = []
    for _ in range(trials):
        with torch.cuda.stream(stream):
            torch.cuda._sleep(1_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
        torch.cuda.synchronize(dev)
        out.append(e0.elapsed_time(e1) / reps)
    return float(statistics.median(out))


def make_line(*, cfg_id, cfg, world, steps, warmup, elapsed_ms, evals_total, pairs_per_launch,
              stage_ms, sm_count, clocks, T_surv, B_local, T_local, P, M_mean, traffic, e2e, cpu,
              reweight_launches=1, b2b_ms=None, reweight_bytes=None, reweight_bytes_b2b=None):
    """The one JSON line of the GPU arm (pure function of the measurements)."""
    f_max = (clocks.get("sm_max_mhz") or 1965.0) * 1e6
    peak = sm_count * COMPAT_PAIRS_PER_CLK_PER_SM * f_max
    peak_sfu = sm_count * SFU_EX2_PER_CLK_PER_SM * f_max
    stage_mean = {n: statistics.mean(v) for n, v in stage_ms.items()}
    achieved = pairs_per_launch / (stage_mean["compat"] * 1e-3)
    hbm = hbm_peak()

    def hbm_kernel(name, nbytes, nbytes_b2b=None):
        nbytes = int(nbytes)
        gbps1 = nbytes / (stage_mean[name] * 1e-3) / 1e9 if stage_mean[name] > 0 else 0.0
        ms = (b2b_ms or {}).get(name)
        if ms is None:   # only the serialised step's single launches were timed
            return {"bound": "hbm", "bytes_per_launch": nbytes, "achieved_GBps": gbps1,
                    "peak_GBps": hbm, "frac": gbps1 / hbm}
        nbytes = int(nbytes_b2b) if nbytes_b2b is not None else nbytes
        gbps = nbytes / (ms * 1e-3) / 1e9
        return {"bound": "hbm", "bytes_per_launch": nbytes, "achieved_GBps": gbps, "peak_GBps": hbm,
                "frac": gbps / hbm, "ms_per_launch": ms,
                "timing": "mean of 10 launches back to back between two events (same inputs)",
                "single_launch_frac": gbps1 / hbm}

    sm_mhz = clocks.get("sm_mhz")
    return {
        "metric": METRIC,
        "value": evals_total / (elapsed_ms * 1e-3),
        "unit": "evals/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": elapsed_ms / steps,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": workload_config(cfg_id, cfg, world, M_mean, evals_total / steps),
        "schedule": "software-pipelined steps: predict + birth of step k into a spare state buffer on a "
                    "high-priority stream beside compat of step k-1, reweight beside compat on a second stream "
                    "(double-buffered state and weights, event-ordered); stages_ms timed in a separate "
                    "serialised pass",
        "roofline": {"bound": "alu", "kernel": "compat (exp: MUFU.EX2 + FMA-pipe polynomial)",
                     "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "Geval/s",
                     "frac": achieved / peak,
                     "peak_basis": f"{sm_count} SM x {COMPAT_PAIRS_PER_CLK_PER_SM:.2f} pairs/clk "
                                   f"({SFU_EX2_PER_CLK_PER_SM} ex2/clk + {FMA_LANES_PER_CLK_PER_SM} FP32 lanes/clk, measured by "
                                   f"glmb_peaks; 5 lanes + 1 exp per pair) x {f_max / 1e6:.0f} MHz",
                     "frac_of_mufu_only_bound": achieved / peak_sfu,
                     "frac_at_measured_clock": (achieved / (sm_count * COMPAT_PAIRS_PER_CLK_PER_SM * sm_mhz * 1e6)
                                                if sm_mhz else None),
                     "traffic": traffic},
        "hbm_kernels": {"predict": hbm_kernel("predict", T_surv * P * 40),
                        "birth": dict(hbm_kernel("birth", B_local * P * 24), bound="launch",
                                      note="3 MB per launch at cfg3 (16 tracks): the launch and its ramp, "
                                           "not HBM, set its time; the fraction is for reference"),
                        "reweight": dict(hbm_kernel("reweight", reweight_bytes if reweight_bytes is not None
                                                    else T_local * P * 16, reweight_bytes_b2b),
                                         bytes_basis="16 B per particle of a track with a measurement (x, y, w "
                                                     "read, w written), 8 B of one without (w copied)")},
        "stages_ms": stage_mean,
        "gpu_launches": ((1 if T_surv else 0) + (1 if B_local else 0) + 1 + reweight_launches) * steps,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": None if cpu is None else
        {k: v for k, v in cpu.items() if k in ("value", "unit", "cores", "kind", "sample", "single_core")},
    }


# ------------------------------------------------------------------ GLMB update
def skip_probe(st, dev, L, reps: int = 10, k_late: int = 0) -> dict:
    """Exact zero-tile skipping (glmb_compat_skipping, opt-in, not the headline): compat dense and
    skipping on the step-0 clouds (a fresh copy of the scene, births drawn) and on the bench's
    own state after its timed steps (diffused clouds), CUDA-event means over `reps` launches;
    evaluated pairs = dense pairs - the device count of skipped pairs, with their rate against
    the same combined exp-pipe bound as the headline; bit-identity of C and the gate words.
    late_state = the bench's particles after its timed and end-to-end steps (diffused clouds)."""
    import torch
    from paper_2512_06230_b200.step import GlmbStep
    fresh = GlmbStep(st.scene, device=dev)
    fresh.birth(0)
    out = {"note": "glmb_compat_skipping: a warp skips a particle tile when all its measurements are >= 200 "
                   "whitened units^2 from the tile's bounding box (contributions exactly +0 on both exp paths); "
                   "opt-in, the headline is the dense pass and counts the dense pairs"}
    sm = L.glmb_sm_count(dev.index or 0)
    for name, g, kz in (("step0", fresh, 0), ("late_state", st, k_late)):
        Z = g.Z[kz % len(g.Z)]   # the measurements of the step the clouds were last predicted to
        M = Z.shape[0]
        c = g.cfg
        Cs, Gs = torch.empty_like(g.out.C_tracks), torch.empty_like(g.out.gate)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for _ in range(2):
            g.compat(0, Z=Z)
            L.glmb_compat_skipping(g.particles, Z, c.R, c.p_d, c.kappa, c.gamma, None, Cs, Gs, cnt)
        torch.cuda.synchronize(dev)
        e[0].record()
        for _ in range(reps):
            g.compat(0, Z=Z)
        e[1].record()
        cnt.zero_()
        e[2].record()
        for _ in range(reps):
            L.glmb_compat_skipping(g.particles, Z, c.R, c.p_d, c.kappa, c.gamma, None, Cs, Gs, cnt)
        e[3].record()
        torch.cuda.synchronize(dev)
        dense_ms, skip_ms = e[0].elapsed_time(e[1]) / reps, e[2].elapsed_time(e[3]) / reps
        pairs = M * g.T_local * g.P
        evaluated = pairs - int(cnt.item()) // reps
        ldg = (M + 31) // 32
        same = bool(torch.equal(Cs[:, :M], g.out.C_tracks[:, :M]) and torch.equal(Gs[:, :ldg], g.out.gate[:, :ldg]))
        peak = sm * COMPAT_PAIRS_PER_CLK_PER_SM * 1.965e9
        out[name] = {"dense_ms": dense_ms, "skip_ms": skip_ms, "speedup": dense_ms / skip_ms,
                     "pairs": pairs, "evaluated_pairs": evaluated, "evaluated_frac": evaluated / pairs,
                     "evaluated_pairs_per_s": evaluated / (skip_ms * 1e-3),
                     "frac_of_combined_bound": evaluated / (skip_ms * 1e-3) / peak,
                     "bit_identical": same}
    del fresh
    return out


def verify_fused_gather(sh, dev, stream) -> bool:
    """Before timing (N > 1): the fused compat + peer-store gather must give every rank
    exactly the C_k / gate words an NCCL all-gather of glmb_compat's local columns gives
    (bit-identical by construction).  All ranks agree on the outcome (all_reduce MIN)."""
    import torch
    import torch.distributed as dist
    from paper_2512_06230_b200 import _lib as L
    st = sh.st
    M = sh.load_measurements(0, stream=stream)
    ok = True
    try:
        with torch.cuda.stream(stream):
            sh._broadcast(M)
            Zk = sh.Z(M)
            for k in (0, 1):                  # both symmetric copies
                sh._compat(st.particles, Zk, k, stream)
                sh.symm.barrier(k, stream)
            L.glmb_compat(st.particles, Zk, st.R, st.cfg.p_d, st.cfg.kappa, st.cfg.gamma, st.out.C_clutter,
                          sh.local_C()[:st.T_local], sh.local_gate()[:st.T_local], stream)
        torch.cuda.synchronize(dev)
        dist.all_gather_into_tensor(sh.gathered, sh.block)
        torch.cuda.synchronize(dev)
        ldg_used = (M + 31) // 32
        for k in (0, 1):
            buf = sh.symm.buffer(k)
            ok &= bool(torch.equal(buf[:, :M], sh.gathered[:, :M]))
            ok &= bool(torch.equal(buf[:, sh.ldc:sh.ldc + ldg_used], sh.gathered[:, sh.ldc:sh.ldc + ldg_used]))
    except Exception as e:  # noqa: BLE001
        print(f"[bench] fused gather check raised {e!r}", file=sys.stderr)
        ok = False
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return bool(flag.item())


def bench_update(a, st, scene, cfg, dev, stream, L, k_last: int):
    """The hypothesis update and particle loop that consume the step's C_k:
    death_prob -> compat_rows -> assoc_sample -> dedup -> prune -> assoc_pairs ->
    reweight_pairs -> resample, on the device-resident C_k / particles of the last timed
    step, H_old x H_up samples, tau = 1e-5, H_max (H_up = 100, tau = 1e-5,
    H_max <= 100).  Reported beside the headline metric (not part of it)."""
    import torch
    from paper_2512_06230_b200.hyp import HypothesisUpdate, ParticleUpdate
    from paper_2512_06230_b200.scenes import hypothesis_inputs
    T = st.T_local
    zi = k_last % len(st.Z)    # the step whose C_k and particles the update consumes
    Z = st.Z[zi]
    M = Z.shape[0]
    pm, plw, ps = hypothesis_inputs(cfg.T, cfg.B, a.h_old, seed=cfg.seed)
    pm_d = torch.from_numpy(pm.view(np.int32)).to(dev)
    plw_d = torch.from_numpy(plw).to(dev)
    ps_d = torch.from_numpy(ps).to(dev)
    hu = HypothesisUpdate(T, st.M_max, a.h_old, a.h_up, a.h_max, device=dev)
    pu = ParticleUpdate(T, st.M_max, a.h_max, st.P, K_cap=16 * T, device=dev)
    names = ["death_prob", "compat_rows", "assoc_sample", "dedup", "prune", "assoc_pairs",
             "reweight_pairs", "resample"]
    stage = {n: [] for n in names}
    total = []

    def run(k, timed):
        evs = {}
        def mark(name):
            if timed:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                evs[name] = e
        with torch.cuda.stream(stream):
            if timed:
                mark("start")
            hu.run(st.out.C_tracks, st.out.gate, M, ps_d, pm_d, plw_d, cfg.p_d, cfg.kappa, 1e-5,
                   seed=cfg.seed, step=k, stream=stream, mark=mark)
            pu.run(st.particles, Z, st.R, hu.keep_idx, a.h_max, hu.alive, hu.theta, M, seed=cfg.seed,
                   step=k, stream=stream, n_hyp_dev=hu.n_kept, mark=mark)
        return evs

    for k in range(a.warmup):
        run(k, False)
    torch.cuda.synchronize(dev)
    all_evs = [run(k, True) for k in range(a.warmup, a.warmup + a.steps)]
    torch.cuda.synchronize(dev)
    for evs in all_evs:
        prev = evs["start"]
        for n in names:
            stage[n].append(prev.elapsed_time(evs[n]))
            prev = evs[n]
        total.append(evs["start"].elapsed_time(evs["resample"]))
    # the same chain as one glmb_update call (the tracker's path: one argument block, the
    # death probabilities and row counts in one grid), timed end to end with two events
    from paper_2512_06230_b200.hyp import update_params
    one = []
    for k in range(a.warmup, a.warmup + a.steps):
        prm = update_params(hu, pu, st.particles, st.out.C_tracks, st.out.gate, M, Z, st.R, ps_d, pm_d, plw_d,
                            cfg.p_d, cfg.kappa, 1e-5, cfg.seed, k, out=pu.out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.glmb_update(prm, stream)
        e1.record(stream)
        one.append((e0, e1))
    torch.cuda.synchronize(dev)
    one_ms = statistics.mean(x.elapsed_time(y) for x, y in one)
    n_kept = int(hu.n_kept.item())
    n_pairs = pu.n_pairs_checked()
    rp = hu.row_ptr[:M + 1].cpu().numpy()
    row_len = np.diff(rp)
    fl = pu.flags[:n_pairs].cpu().numpy()
    n_res = int(((fl >> 1) & 1).sum())
    stage_mean = {n: statistics.mean(v) for n, v in stage.items()}
    P = st.P
    hbm = hbm_peak()

    def hbm_stage_ms(nbytes, ms):
        gbps = nbytes / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        return {"bytes": int(nbytes), "achieved_GBps": gbps, "peak_GBps": hbm, "frac": gbps / hbm, "ms_per_launch": ms}

    def hbm_stage(name, nbytes):
        return hbm_stage_ms(nbytes, stage_mean[name])

    # algorithmic bytes: reweight_pairs reads x, y, w and writes w' (16 B per particle and
    # pair); resample reads w' (4 B) and, per resampled pair, gathers 5 state fields (20 B)
    # and writes 6 (24 B), per kept pair copies 6 fields (24 + 24 B)
    plen = np.diff(pu.pair_ptr[:n_pairs + 1].cpu().numpy()) if n_pairs else np.zeros(0, np.int64)
    rp_bytes = P * (16 * int((plen > 0).sum()) + 8 * int((plen == 0).sum()))
    hbm_f2 = {"reweight_pairs": hbm_stage("reweight_pairs", rp_bytes),
              "resample": hbm_stage("resample", P * (4 * n_pairs + 44 * n_res + 48 * (n_pairs - n_res)))}
    # the pair update again, 10 launches back to back on the last update's pair lists (idempotent:
    # reads the predicted particles, writes w_new); the headline frac, the single launch beside it
    K = min(pu.K_cap, max(1, a.h_max * T))
    rp_call = lambda: L.glmb_reweight_pairs(st.particles, Z, st.R, K, pu.n_pairs, pu.pair_track, pu.pair_ptr,  # noqa: E731
                                            pu.pair_meas, pu.w_new[:K], pu.log_norm, pu.flags, pu.ess, stream)
    ms_rp = stage_mean["reweight_pairs"] if a.no_b2b else back_to_back_ms(rp_call, stream, dev)
    rp_single = hbm_f2["reweight_pairs"]["frac"]
    hbm_f2["reweight_pairs"] = dict(hbm_stage_ms(rp_bytes, ms_rp), single_launch_frac=rp_single,
                                    pairs_without_measurement=int((plen == 0).sum()),
                                    timing="single launches (--no-b2b)" if a.no_b2b else
                                    "mean of 10 launches back to back between two events (same inputs)")
    # the two-stage sampler's bound (R24): one Philox4x32-10 block per (sample, parent track quad)
    # and per (sample, row quad holding a parent entry) -- 10 rounds of 2 IMAD.WIDE.U32 (FMA-heavy
    # pipe, 64 lanes/clk/SM) and 2 LOP3 (ALU pipe, 64 lanes/clk/SM), the two pipes in parallel --
    # against the theta / alive / log-weight / fingerprint writes at the HBM peak
    col = hu.col[:int(rp[-1])].cpu().numpy()
    row_of = np.repeat(np.arange(M), row_len)
    ldt = pm.shape[1]
    blocks = 0
    for h in range(a.h_old):
        bits = np.zeros(32 * ldt, bool)
        bits[:] = np.unpackbits(pm[h].astype("<u4").view(np.uint8), bitorder="little").astype(bool)
        bits[T:] = False
        tq = int(bits[:(T + 3) // 4 * 4].reshape(-1, 4).any(axis=1).sum())
        rows_h = np.unique(row_of[bits[col]] // 4) if len(col) else np.zeros(0)
        blocks += a.h_up * (tq + len(rows_h))
    f_clk = 1.965e9
    sm = L.glmb_sm_count(dev.index or 0)
    alu_s = blocks * 20.0 / (64.0 * sm * f_clk)
    n_s = a.h_old * a.h_up
    bytes_s = n_s * (4 * M + 4 * ldt + 8 + 8)
    hbm_s = bytes_s / (hbm * 1e9)
    t_s = stage_mean["assoc_sample"] * 1e-3
    sampler = {"philox_blocks": blocks, "alu_bound_us": alu_s * 1e6, "bytes_written": bytes_s,
               "hbm_bound_us": hbm_s * 1e6, "bound": "hbm" if hbm_s >= alu_s else "alu",
               "frac": max(alu_s, hbm_s) / t_s,
               "basis": "Philox: 20 IMAD.WIDE + 20 LOP3 per block on two 64-lane/clk/SM pipes; theta, alive, "
                        "log-weight and fingerprint bytes at the measured HBM peak"}
    return {"workload": f"cfg{a.config if a.config is not None else 3} C_k (T_k={T}, M={M}) + particles; "
                        f"H_old={a.h_old} x H_up={a.h_up}, tau=1e-5, H_max={a.h_max} (P:186)",
            "ms": statistics.mean(total), "one_call_ms": one_ms, "stages_ms": stage_mean, "hbm_kernels": hbm_f2,
            "assoc_sample_roofline": sampler,
            "n_samples": a.h_old * a.h_up, "n_unique": int(hu.unique.sum().item()), "n_kept": n_kept,
            "n_pairs": n_pairs, "n_resampled": n_res,
            "gated_entries": int(rp[-1]), "row_len_max": int(row_len.max()) if M else 0,
            "rows_empty": int((row_len == 0).sum()),
            "gpu_launches_per_update": 14,
            "note": "device-resident; no host round trip inside (device counts n_kept / n_pairs)"}


# ------------------------------------------------------------------ configs 0-2 (launch-bound): CUDA graphs
def bench_graphs(dev, reps: int = 200):
    """the small configs are launch-bound; one whole step (glmb_step: predict,
    birth, compat, reweight) is captured once in a CUDA graph and replayed.  Reports us/step
    eager (four C-ABI launches from Python) and replayed, and the replayed evals/s."""
    import torch
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    out = {}
    for cfg_id in (0, 1, 2):
        scene = make_scene(cfg_id, steps=1)
        st = GlmbStep(scene, device=dev)
        s = torch.cuda.Stream(device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            for _ in range(3):
                st.run(0, s)
            s.synchronize()
            e0.record(s)
            for _ in range(reps):
                st.run(0, s)
            e1.record(s)
            s.synchronize()
            eager = e0.elapsed_time(e1) / reps
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                st.run(0, s)
            for _ in range(3):
                g.replay()
            s.synchronize()
            e0.record(s)
            for _ in range(reps):
                g.replay()
            e1.record(s)
            s.synchronize()
            replay = e0.elapsed_time(e1) / reps
        evals = st.evals(0)
        out[f"cfg{cfg_id}"] = {"T_k": st.T_local, "P": st.P, "M": len(scene.Z[0]), "evals_per_step": evals,
                               "us_per_step_eager": eager * 1e3, "us_per_step_graph": replay * 1e3,
                               "evals_per_s_graph": evals / (replay * 1e-3)}
    return out


# ------------------------------------------------------------------ the paper's convoy
def bench_convoy(dev, seeds=range(10)):
    """The paper's own benchmark shape: N = 20 objects, D = 5, sigma = 0.25, delta = 2,
    H_up = 100, tau = 1e-5, H_max = 100, 548 updates, through tracker.ConvoyTracker (every stage a
    libglmb kernel; the host copies Z_k in and reads one count per update).  The paper's protocol
    (P:186): 10 runs (seeds 0-9), reported as mean +- SEM over the runs.  Per-update time is
    wall clock around the whole update (what the paper's 0.1 s real-time line refers to),
    plus the device time between the first and last kernel; accuracy by P:213-215's metrics."""
    from paper_2512_06230_b200.scenes import ConvoyConfig
    from paper_2512_06230_b200.tracker import convoy_metrics, run_convoy
    run_convoy(ConvoyConfig(N=2, H_max=10, K=20), K_cap=256, device=dev)     # warm-up (module load, allocator)
    per_seed = []
    wall_all, dev_all = [], []
    for sd in seeds:
        cfg = ConvoyConfig(N=20, H_max=100, seed=sd)
        recs, ests, truth = run_convoy(cfg, K_cap=4096, device=dev)
        card, dist = convoy_metrics(ests, truth)
        wall = np.array([r.wall_ms for r in recs])
        devms = np.array([r.device_ms for r in recs])
        wall_all.append(wall)
        dev_all.append(devms)
        per_seed.append({"seed": sd, "card_err": card, "track_err_m": dist, "update_ms_mean": float(wall.mean()),
                         "device_ms_mean": float(devms.mean()), "pairs_max": max(r.n_pairs for r in recs)})
    stages = {}
    run_convoy(ConvoyConfig(N=20, H_max=100, seed=0), K_cap=4096, device=dev, with_estimates=False,
               stage_ms=stages)   # per-stage pass
    wall, devms = np.concatenate(wall_all), np.concatenate(dev_all)
    mse = lambda key: (float(np.mean([p[key] for p in per_seed])),
                       float(np.std([p[key] for p in per_seed], ddof=1) / np.sqrt(len(per_seed))))
    card_m, card_sem = mse("card_err")
    dist_m, dist_sem = mse("track_err_m")
    return {"workload": "convoy N=20, D=5, sigma=0.25 m, delta=2, lambda=0, H_up=100, tau=1e-5, H_max=100, "
                        f"548 updates (P:182-186; synthetic figure-eight ground track, R35); {len(per_seed)} runs "
                        "(seeds), mean +- SEM (P:186)",
            "update_ms_mean": float(wall.mean()), "update_ms_p95": float(np.percentile(wall, 95)),
            "update_ms_max": float(wall.max()), "device_ms_mean": float(devms.mean()),
            "realtime_budget_ms": 100.0,
            "card_err_mean": card_m, "card_err_sem": card_sem,
            "track_err_m_mean": dist_m, "track_err_m_sem": dist_sem,
            "per_seed": per_seed,
            "stages_ms": stages, "stages_note": "seed 0, a second pass with a CUDA event after every stage",
            "paper": "L40S: 'under the threshold of 0.1 seconds per update ... almost always' (P:211), "
                     "card. error low at H_max=100, matched error < 0.15 m (P:213-215)"}


# ------------------------------------------------------------------ GPU arm
def main():
    a = parse()
    rank, world, local = dist_env()
    cfg_id = a.config if a.config is not None else (3 if world == 1 else 4)
    if a.impl == "reference":
        return reference_arm(a, cfg_id)

    import torch
    import torch.distributed as dist
    from paper_2512_06230_b200 import _lib as L
    from paper_2512_06230_b200.build import build
    from paper_2512_06230_b200.scenes import CONFIGS, make_scene
    from paper_2512_06230_b200.dist import ShardedStep
    from paper_2512_06230_b200.step import GlmbStep, PipelinedSteps

    # GLMB_BENCH_BACKEND=gloo (test hook): the N > 1 path with gloo collectives on host-staged
    # copies, ranks mapped onto the available GPUs -- a dry run of this code path on a box
    # with fewer GPUs than ranks (the kernels of the ranks never wait on each other)
    backend = os.environ.get("GLMB_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local)   # before NCCL init: each rank's communicator binds its own GPU
    if rank == 0:
        build()
    coll_dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")

    def barrier():
        if backend == "nccl":
            dist.barrier(device_ids=[local])
        else:
            dist.barrier()
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        barrier()
        build()  # no-op once rank 0 has built
    L.glmb_init(local)
    dev = torch.device("cuda", local)
    cfg = CONFIGS[cfg_id]
    # Every executed step k uses the scene's own Z_k, theta_k (the truth moves on with the
    # predicted clouds): the timed loop runs steps [0, W + K), the serialised per-kernel pass
    # [W + K, W + 2K), the end-to-end legs (W + K) each after that -- the sequence is generated
    # that long (prefix-stable: step k's data do not depend on the length), past BASELINE's
    # own step count where that is shorter.
    k_iso = a.warmup + a.steps                  # first step of the serialised pass
    k_e2e = k_iso + a.steps                     # first step of the end-to-end legs
    n_steps_scene = max(cfg.steps, k_e2e + 2 * (a.warmup + a.steps))
    stream = torch.cuda.Stream(device=dev)
    side = torch.cuda.Stream(device=dev)   # reweight overlaps compat (double-buffered weights)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    sh = None
    gather = "none (one rank)"
    if world > 1:
        # W > 1 (dist.ShardedStep): Z_k / theta_k live on rank 0 and are broadcast inside the
        # timed region (one packed collective); survivors and births split evenly over the
        # ranks; C_k's column blocks + gate words all-gathered (one collective) with the
        # log-normalisers and flags -- or, fused, stored by compat into every rank's
        # symmetric-memory copy over NVLink (GLMB_FUSED_GATHER=0: NCCL all-gather)
        fused = os.environ.get("GLMB_FUSED_GATHER", "1") != "0" and backend == "nccl"
        try:
            sh = ShardedStep(cfg_id, device=dev, steps=n_steps_scene, fused=fused,
                             stage_on_host=backend != "nccl")
        except Exception as e:  # noqa: BLE001
            if not fused:
                raise
            print(f"[bench] symmetric memory unavailable ({e}); NCCL all-gather", file=sys.stderr)
            sh = ShardedStep(cfg_id, device=dev, steps=n_steps_scene, fused=False)
        gather = ("fused: compat stores its columns into every rank's symmetric-memory C_k (NVLink), device barrier"
                  if sh.symm is not None else "NCCL all_gather_into_tensor of the column blocks"
                  if backend == "nccl" else "gloo all_gather of host-staged column blocks (dry-run test hook)")
        st, scene = sh.st, sh.scene
    else:
        scene = make_scene(cfg_id, steps=n_steps_scene)
        st = GlmbStep(scene, device=dev)
    stage_names = ["predict", "birth", "compat", "reweight"]
    stage_ms = {n: [] for n in stage_names}

    # N = 1: software-pipelined steps (step.PipelinedSteps): predict + birth of step k into the
    # spare state buffer on a high-priority stream beside compat of step k-1, reweight beside compat
    pipe = PipelinedSteps(st, stream, side) if sh is None else None

    def one_step(k):
        """One step as timed (PipelinedSteps at N = 1); at W > 1 the broadcast, the four calls
        and the gather in order (ShardedStep.step, reweight beside compat)."""
        if sh is not None:
            M = sh.load_measurements(k, stream=stream)
            sh.step(k, M, stream=stream, side=side)
            return
        pipe.step(k)

    def join_streams():
        """The timed region ends when every stream's last step work is done."""
        if pipe is not None:
            pipe.join()

    def isolated_step(k):
        """The same four calls serialised on `stream`, with an event between each, so
        every kernel's own launch duration is measured (the overlapped step hides
        reweight behind compat, so its events there would time the overlap)."""
        zi = k % len(st.Z)
        marks = [ev() for _ in range(5)]
        with torch.cuda.stream(stream):
            marks[0].record(stream)
            st.predict(k, stream)
            marks[1].record(stream)
            st.birth(k, stream)
            marks[2].record(stream)
            st.compat(k, stream)
            marks[3].record(stream)
            st.reweight(k, stream, out_of_place=True)
            marks[4].record(stream)
        return marks

    for k in range(a.warmup):
        one_step(k)
    torch.cuda.synchronize(dev)
    if sh is not None and sh.symm is not None and not verify_fused_gather(sh, dev, stream):
        sh.symm = None   # every rank falls back together (collective decision)
        gather = "NCCL all_gather_into_tensor of the column blocks (fused gather failed its check)"
        print("[bench] fused gather disagreed with the NCCL all-gather; using NCCL", file=sys.stderr)
    sampler = ClockSampler(local)
    if world > 1:
        barrier()
    torch.cuda.synchronize(dev)
    t_start, t_end = ev(), ev()
    step_marks = []
    with sampler:
        t_start.record(stream)
        if pipe is not None:
            pipe.start_after(t_start)
        for k in range(a.warmup, a.warmup + a.steps):
            one_step(k)
            e = ev()
            e.record(stream)
            step_marks.append(e)
        join_streams()
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    per_step = [(step_marks[0] if i == 0 else step_marks[i - 1]).elapsed_time(step_marks[i]) if i else
                t_start.elapsed_time(step_marks[0]) for i in range(len(step_marks))]
    if world > 1:
        barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    # per-kernel durations: the same steps again, serialised (outside the timed region)
    all_marks = [isolated_step(k) for k in range(k_iso, k_e2e)]
    torch.cuda.synchronize(dev)
    for m in all_marks:
        for n, (m0, m1) in zip(stage_names, zip(m[:-1], m[1:])):
            stage_ms[n].append(m0.elapsed_time(m1))
    b2b = None if a.no_b2b else hbm_back_to_back(st, stream, dev, k_e2e - 1)
    evals_local = sum(st.evals(k) for k in range(a.warmup, a.warmup + a.steps))
    pairs_local = sum(len(scene.Z[k % len(scene.Z)]) * st.T_local * st.P
                      for k in range(a.warmup, a.warmup + a.steps))
    if world > 1:
        t = torch.tensor([elapsed_ms, float(evals_local)], dtype=torch.float64, device=coll_dev)
        tmax = t.clone(); dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        tsum = t.clone(); dist.all_reduce(tsum[1:], op=dist.ReduceOp.SUM)
        elapsed_ms, evals_total = float(tmax[0]), float(tsum[1])
    else:
        evals_total = float(evals_local)

    # ---- the hypothesis update on this step's C_k (before the e2e legs step the particles on)
    update = None
    if world == 1 and not a.no_update:
        update = bench_update(a, st, scene, cfg, dev, stream, L, k_e2e - 1)

    # ---- launch-bound small configs: one whole step (glmb_step) captured in a CUDA graph
    graphs = None
    if world == 1 and not a.no_graphs:
        graphs = bench_graphs(dev)

    # ---- end to end through the public C-ABI entry with host buffers (N=1 leg per rank)
    e2e = None
    if not a.no_e2e:
        M_max = st.M_max
        pin = lambda t: t.pin_memory()
        Zh = [pin(torch.from_numpy(z)) for z in scene.Z]
        thh = [pin(torch.from_numpy(t)) for t in scene.theta]
        Zd = torch.empty(M_max, 2, device=dev)
        thd = torch.empty(M_max, dtype=torch.int32, device=dev)
        o = st.out
        Cc_h = pin(torch.empty(M_max))
        Ct_h = pin(torch.empty(st.T_local, st.ldc))
        G_h = pin(torch.empty(st.T_local, st.ldg, dtype=torch.int32))
        ln_h = pin(torch.empty(st.T_local))
        fl_h = pin(torch.empty(st.T_local, dtype=torch.int32))
        copy_stream = torch.cuda.Stream(device=dev)   # dense read-back of C_k overlapping reweight
        cap = st.T_local * M_max                       # device CSR capacity (never overflows)
        rp_d = torch.empty(M_max + 1, dtype=torch.int32, device=dev)
        col_d = torch.empty(cap, dtype=torch.int32, device=dev)
        val_d = torch.empty(cap, dtype=torch.float32, device=dev)
        lv_d = torch.empty(cap, dtype=torch.float64, device=dev)
        first_h = 4 * M_max                            # the speculative first copy (entries); a second,
                                                       # exact copy if the gated entries exceed it
        rp_h = pin(torch.empty(M_max + 1, dtype=torch.int32))
        col_h = pin(torch.empty(cap, dtype=torch.int32))   # host capacity = the device capacity
        val_h = pin(torch.empty(cap))

        def host_step_csr(k):
            """C_k read back as the CSR of its gated entries (glmb_step_host_csr)."""
            zi = k % len(Zh)
            nnz = L.glmb_step_host_csr(st.step_params(k, out_of_place=True), Zh[zi], thh[zi], Zd, thd,
                                       o.C_tracks, o.gate, o.log_norm, o.flags, rp_d, col_d, val_d, lv_d, rp_h,
                                       col_h, val_h, ln_h, fl_h, stream, aux_stream=copy_stream, first_copy=first_h)
            st.swap_weights()
            M = Zh[zi].shape[0]
            first = min(first_h, cap)                  # entries copied speculatively, then the rest
            return M * 12, (M + 1) * 4 + max(first, nnz) * 8 + st.T_local * 8

        def host_step_dense(k):
            """C_k read back dense (glmb_step_host)."""
            zi = k % len(Zh)
            L.glmb_step_host(st.step_params(k), Zh[zi], thh[zi], Zd, thd, o.C_clutter,
                             o.C_tracks, o.gate, o.log_norm, o.flags, Cc_h, Ct_h, G_h, ln_h, fl_h, stream,
                             copy_stream)
            M = Zh[zi].shape[0]
            return M * 12, M * 4 + st.T_local * st.ldc * 4 + st.T_local * st.ldg * 4 + st.T_local * 8

        def timed(fn, k0):
            """W warm-up then K timed steps of the leg from scene step k0; returns the seconds,
            the bytes per step and the whole job's evals of the timed steps."""
            h2d = d2h = 0
            for k in range(k0, k0 + a.warmup):
                fn(k)
            if world > 1:
                barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for k in range(k0 + a.warmup, k0 + a.warmup + a.steps):
                hb, db = fn(k)
                h2d += hb
                d2h += db
            sec = time.perf_counter() - t0
            ev_loc = float(sum(st.evals(k) for k in range(k0 + a.warmup, k0 + a.warmup + a.steps)))
            if world > 1:
                t = torch.tensor([sec, ev_loc], dtype=torch.float64, device=coll_dev)
                tmax = t.clone(); dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
                tsum = t.clone(); dist.all_reduce(tsum[1:], op=dist.ReduceOp.SUM)
                sec, ev_loc = float(tmax[0]), float(tsum[1])
            return sec, h2d // a.steps, d2h // a.steps, ev_loc

        def host_step_dist(k):
            """W > 1: ShardedStep.step_host_csr -- rank 0's pinned Z_k / theta_k H2D, the broadcast,
            every rank's shard, the gathers, and rank 0's CSR read-back of the gathered C_k."""
            zi = k % len(Zh)
            _, hb, db = sh.step_host_csr(k, Zh[zi], thh[zi], stream=stream, side=side)
            return hb, db

        if sh is not None:
            e2e_s, h2d, d2h, e2e_ev = timed(host_step_dist, k_e2e)
            e2e = {"value": e2e_ev / e2e_s, "unit": "evals/s",
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                   "ms_per_step": e2e_s * 1e3 / a.steps,
                   "note": "dist.ShardedStep.step_host_csr: rank 0's pinned H2D of Z_k, theta_k; the broadcast; "
                           "every rank's predict/birth/compat/reweight; the C_k + gate all-gather (or fused peer "
                           "stores) and the log_norm/flags gather; rank 0 builds the CSR of the gathered C_k and "
                           "reads it back with log_norm and flags; synchronised each step; max over ranks"}
    if not a.no_e2e and sh is None:
        e2e_s, h2d, d2h, e2e_ev = timed(host_step_csr, k_e2e)
        dn_s, dn_h2d, dn_d2h, dn_ev = timed(host_step_dense, k_e2e + a.warmup + a.steps)
        e2e = {"value": e2e_ev / e2e_s, "unit": "evals/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_s * 1e3 / a.steps,
               "note": "glmb_step_host_csr: pinned H2D of Z_k, theta_k; the step (reweight into the spare "
                       "weights beside compat); C_k's gated entries as CSR (row_ptr, col, val) + log_norm, "
                       "flags D2H; synchronised each step; particle state resident on the device",
               "dense": {"value": dn_ev / dn_s, "ms_per_step": dn_s * 1e3 / a.steps,
                         "h2d_bytes_per_step": dn_h2d, "d2h_bytes_per_step": dn_d2h,
                         "note": "glmb_step_host: the same with C_k and the gate words read back dense "
                                 "(on a copy stream overlapping reweight)"}}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    convoy = None
    if world == 1 and not a.no_convoy:
        convoy = bench_convoy(dev)
    skipped = None
    if world == 1 and not a.no_skip_probe:
        k_done = k_e2e + (0 if a.no_e2e else (a.warmup + a.steps) * (1 if sh is not None else 2)) - 1
        skipped = skip_probe(st, dev, L, k_late=k_done if not a.no_e2e else k_e2e - 1)

    cpu = None
    if world == 1 and not a.no_cpu_baseline:
        cpu = oracle_sample(cfg_id, a.cpu_seconds, host_cores())
    Ms = [len(scene.Z[k % len(scene.Z)]) for k in range(a.warmup, a.warmup + a.steps)]
    line = make_line(
        cfg_id=cfg_id, cfg=cfg, world=world, steps=a.steps, warmup=a.warmup,
        elapsed_ms=elapsed_ms, evals_total=evals_total, pairs_per_launch=pairs_local / a.steps,
        stage_ms=stage_ms, sm_count=L.glmb_sm_count(local), clocks=sampler.summary(),
        T_surv=st.T_surv, B_local=st.B_local, T_local=st.T_local, P=st.P, M_mean=float(np.mean(Ms)),
        traffic=compat_traffic(st.T_local, st.P, len(scene.Z[0])), e2e=e2e, cpu=cpu,
        reweight_launches=1 if st.contiguous else 2, b2b_ms=b2b,
        reweight_bytes=statistics.mean(reweight_bytes(st, k) for k in range(k_iso, k_e2e)),
        reweight_bytes_b2b=reweight_bytes(st, k_e2e - 1))
    line["gather"] = gather
    if world > 1:
        line["schedule"] = ("per step: the packed Z_k/theta_k broadcast, predict, birth, compat with reweight "
                            "beside it on a second stream, the C_k/gate and log_norm gathers")
    line["ms_per_step_p50"] = float(np.percentile(per_step, 50))
    line["ms_per_step_p95"] = float(np.percentile(per_step, 95))
    if graphs is not None:
        line["small_configs_graph"] = graphs
    if update is not None:
        line["glmb_update"] = update
    if convoy is not None:
        line["convoy"] = convoy
    if skipped is not None:
        line["compat_exact_skip"] = skipped
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
