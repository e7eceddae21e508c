"""Dev probe: cfg2 multi-index builds with wall-clock timing (and for ncu captures of build kernels)."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import time
import paper_1712_06326_b200 as zb
import workloads
img, kn, p = workloads.cfg2()
t = time.perf_counter()
ctx = zb.Context()
print("ctx s", time.perf_counter() - t)
for i in range(3):
    t = time.perf_counter()
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=11, dims=12), ctx=ctx)
    print("build", i, "wall s", round(time.perf_counter() - t, 4), "event ms", round(mi.info.build_seconds * 1e3, 3))
t = time.perf_counter()
mi.rebuild()
print("rebuild wall s", round(time.perf_counter() - t, 4), "event ms", round(mi.info.build_seconds * 1e3, 3))
