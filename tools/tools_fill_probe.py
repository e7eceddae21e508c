"""dev probe: cfg2 fill loop with per-part timing (ZI_DEBUG_QUERY)."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import time

import paper_1712_06326_b200 as zb
import workloads

img, kn, p = workloads.cfg2()
mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=11, dims=12, knn=80))
t = time.perf_counter()
out, recs, st = mi.inpaint()
print("iterations", st.iterations, "seconds", time.perf_counter() - t)
