#!/usr/bin/env python
"""Timeline of step.PipelinedSteps at cfg3 (diagnostic): CUDA events around each predict (pred
stream), reweight (side) and compat (main); prints their start/end in ms from the first event,
to see whether predict_k runs inside compat_{k-1}."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2512_06230_b200 import _lib as L  # noqa: E402
from paper_2512_06230_b200.scenes import make_scene  # noqa: E402
from paper_2512_06230_b200.step import GlmbStep, PipelinedSteps  # noqa: E402

torch.cuda.set_device(0)
L.glmb_init(0)
st = GlmbStep(make_scene(int(sys.argv[1]) if len(sys.argv) > 1 else 3, steps=1), device="cuda:0")
main, side = torch.cuda.Stream(), torch.cuda.Stream()
pipe = PipelinedSteps(st, main, side)
E = lambda: torch.cuda.Event(enable_timing=True)
orig_pred, orig_rw, orig_compat = st.predict_to_spare, st.reweight, L.glmb_compat
marks = []


def wrap(name, fn, stream_of):
    def f(*a, **kw):
        s = stream_of(*a, **kw)
        e0, e1 = E(), E()
        e0.record(s)
        r = fn(*a, **kw)
        e1.record(s)
        marks.append((name, e0, e1))
        return r
    return f


st.predict_to_spare = wrap("predict", orig_pred, lambda k, stream: stream)
st.reweight = wrap("reweight", orig_rw, lambda k, stream, **kw: stream)
L.glmb_compat = wrap("compat", orig_compat, lambda *a: a[-1])
for k in range(3):
    pipe.step(k)
torch.cuda.synchronize()
marks.clear()
t0 = E()
t0.record(main)
for k in range(3, 9):
    pipe.step(k)
pipe.join()
torch.cuda.synchronize()
for name, e0, e1 in marks:
    print(f"{name:9s} {t0.elapsed_time(e0):8.3f} -> {t0.elapsed_time(e1):8.3f}")
