#!/usr/bin/env python
"""A/B sweep of glmb_compat launch knobs at a BASELINE config (GPU box only).

    python profiles/compat_sweep.py [--config 3] [--reps 10] SETTING [SETTING ...]

SETTING is "K,EMU[,EMU_FOLD[,PRED]]" (GLMB_COMPAT_K, GLMB_COMPAT_EMU,
GLMB_COMPAT_EMU_FOLD; PRED predict steps before timing: the scene's clouds
widen with every predict, so PRED = 0 times compact clouds (folded tiles) and
PRED = 25 the bench's late steps (exact-difference tiles).  Each setting runs in its
own process (the knobs are read once per process) and prints one JSON line:
mean compat launch time over `reps` launches (CUDA events), pairs/s and
pairs/clk/SM at the sampled clock.  Diagnostics only -- not a bench number.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg_id: int, reps: int, n_pred: int = 0):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2512_06230_b200 import _lib as L
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    torch.cuda.set_device(0)
    L.glmb_init(0)
    s = make_scene(cfg_id, steps=1)
    st = GlmbStep(s, device="cuda:0")
    for k in range(n_pred):
        st.predict(k)
    st.birth(0)
    for _ in range(3):
        st.compat(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        st.compat(0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pairs = len(s.Z[0]) * st.T_local * st.P
    sm = L.glmb_sm_count(0)
    print(json.dumps({"K": os.environ.get("GLMB_COMPAT_K"), "EMU": os.environ.get("GLMB_COMPAT_EMU"),
                      "EMU_FOLD": os.environ.get("GLMB_COMPAT_EMU_FOLD"), "pred": n_pred,
                      "ms": ms, "pairs_per_s": pairs / ms * 1e3,
                      "pairs_per_clk_sm_at_1965": pairs / ms * 1e3 / (sm * 1.965e9)}), flush=True)


def main():
    args = sys.argv[1:]
    if args and args[0] == "--child":
        return child(int(args[1]), int(args[2]), int(args[3]))
    cfg, reps = 3, 10
    if "--config" in args:
        i = args.index("--config"); cfg = int(args[i + 1]); del args[i:i + 2]
    if "--reps" in args:
        i = args.index("--reps"); reps = int(args[i + 1]); del args[i:i + 2]
    for setting in args:
        f = setting.split(",") + ["-4", "0"]
        k, emu, emuf, pred = f[0], f[1], f[2], f[3]
        env = dict(os.environ, GLMB_COMPAT_K=k, GLMB_COMPAT_EMU=emu, GLMB_COMPAT_EMU_FOLD=emuf)
        subprocess.run([sys.executable, __file__, "--child", str(cfg), str(reps), pred], env=env, check=False)


if __name__ == "__main__":
    main()
