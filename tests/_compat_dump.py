"""Helper for the exact-skip tests: glmb_compat on a scene's first step, C, the gate words and
the exact fp32 inputs (x, y, w) saved to an .npz (run in a child process, so environment knobs
read once per process -- GLMB_COMPAT_SKIP -- apply).

    _compat_dump.py cfg n_rows n_pred out [n_cols]

n_cols > n_rows appends that many birth columns (glmb_birth at step 0) after the survivors."""
import sys

import numpy as np


def main(cfg_id: int, n_rows: int, n_pred: int, out: str, n_cols: int = -1) -> None:
    import torch
    from paper_2512_06230_b200 import _lib as L
    from paper_2512_06230_b200.build import build
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    build()
    torch.cuda.set_device(0)
    L.glmb_init(0)
    n_cols = n_rows if n_cols < 0 else n_cols
    s = make_scene(cfg_id, rows=range(0, n_rows), steps=1)
    st = GlmbStep(s, cols=range(0, n_cols), device="cuda:0")
    for k in range(n_pred):
        st.predict(k)
    st.birth(0)
    st.compat(0)
    torch.cuda.synchronize()
    M = len(s.Z[0])
    d = st.particles.data.cpu().numpy()
    np.savez(out, C=st.out.C_tracks.cpu().numpy()[:, :M], G=st.out.gate.cpu().numpy(),
             x=d[0], y=d[1], w=d[5])


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4],
         int(sys.argv[5]) if len(sys.argv) > 5 else -1)
