"""Eager vs CUDA-graph replay of one whole step (tables, bins, fused superpose/inverse/quantise) for C1-C3:
checks the replay is bit-identical and times both (wall clock over 20 steps, one sync at the end)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_1708_04233_b200 as W
from inputs import CONFIGS, make_points
for name in ("C1", "C2", "C3"):
    cfg = CONFIGS[name]
    pts = make_points(cfg)
    p = W.Params.from_config(cfg)
    pl = W.Pipeline(p, len(pts), 0, p.n_h)
    d = torch.from_numpy(pts).cuda()
    s = torch.cuda.Stream()
    pl.stream = s
    with torch.cuda.stream(s):
        pl.run(d); pl.run(d)
    torch.cuda.synchronize()
    ref_bits = pl.bits.clone(); ref_u = pl.field.clone()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            pl.run(d)
    except Exception as e:
        print(name, "capture failed:", repr(e)[:300]); continue
    torch.cuda.synchronize()
    pl.bits.zero_(); pl.field.zero_()
    g.replay(); torch.cuda.synchronize()
    ok = torch.equal(pl.bits, ref_bits) and torch.equal(pl.field, ref_u)
    def t(fn, n=20):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(n): fn()
        torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
    with torch.cuda.stream(s):
        te = t(lambda: pl.run(d))
    tg = t(lambda: g.replay())
    print(f"{name}: graph replay identical={ok}; eager {te:.3f} ms/step, graph {tg:.3f} ms/step (wall, incl. sync)")
