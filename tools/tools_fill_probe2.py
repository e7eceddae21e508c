"""dev probe: fill loop after repeated rebuilds and an e2e-style build/destroy loop (bench order)."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import time
import paper_1712_06326_b200 as zb
import workloads
img, kn, p = workloads.cfg2()
ctx = zb.Context()
mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=11, dims=12, knn=80), ctx=ctx)
t = time.perf_counter(); out, recs, st = mi.inpaint(); print("fresh", round(time.perf_counter() - t, 3))
for _ in range(20):
    mi.rebuild()
t = time.perf_counter(); out, recs, st = mi.inpaint(); print("after rebuilds", round(time.perf_counter() - t, 3))
for _ in range(10):
    m2 = zb.MultiIndex(img, kn, zb.index_config(patch_size=11, dims=12, knn=80), ctx=ctx)
    del m2
t = time.perf_counter(); out, recs, st = mi.inpaint(); print("after e2e builds", round(time.perf_counter() - t, 3))
