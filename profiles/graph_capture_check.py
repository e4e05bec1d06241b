import sys, torch
sys.path.insert(0, '.')
from paper_2512_06230_b200 import _lib as L
from paper_2512_06230_b200.build import build
build(); L.glmb_init(0)
from paper_2512_06230_b200.scenes import make_scene
from paper_2512_06230_b200.step import GlmbStep
st = GlmbStep(make_scene(1, steps=1), device="cuda:0")
s = torch.cuda.Stream()
for name, fn in [("predict", lambda: st.predict(0, s)), ("birth", lambda: st.birth(0, s)),
                 ("compat", lambda: st.compat(0, s)), ("reweight", lambda: st.reweight(0, s)),
                 ("run", lambda: st.run(0, s))]:
    with torch.cuda.stream(s):
        fn(); s.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            fn()
        g.replay(); torch.cuda.synchronize()
        print(name, "OK")
    except Exception as e:
        print(name, "FAIL", str(e).splitlines()[0][:200])
        torch.cuda.synchronize()
