"""Helper for test_compat_exact_skip: glmb_compat on a scene's first step, C and gate saved
to an .npz (run in a child process, so environment knobs read once per process apply)."""
import sys

import numpy as np


def main(cfg_id: int, n_rows: int, n_pred: int, out: str) -> None:
    import torch
    from paper_2512_06230_b200 import _lib as L
    from paper_2512_06230_b200.build import build
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    build()
    torch.cuda.set_device(0)
    L.glmb_init(0)
    s = make_scene(cfg_id, rows=range(0, n_rows), steps=1)
    st = GlmbStep(s, cols=range(0, n_rows), device="cuda:0")
    for k in range(n_pred):
        st.predict(k)
    st.compat(0)
    torch.cuda.synchronize()
    M = len(s.Z[0])
    np.savez(out, C=st.out.C_tracks.cpu().numpy()[:, :M], G=st.out.gate.cpu().numpy())


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
