"""Dev probe: phase clocks of k_pca on cfg2 (ZI_DEBUG_PCA=1) and build timing."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os, time
os.environ.setdefault("ZI_DEBUG_PCA", "1")
import numpy as np
import paper_1712_06326_b200 as zb
import workloads
img, kn, p = workloads.cfg2()
mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=11, dims=12))
print("pca_on_device", mi.info.pca_on_device, "build ms", mi.info.build_seconds * 1e3)
for _ in range(3):
    mi.rebuild()
    print("build ms", mi.info.build_seconds * 1e3, "eigen s", mi.info.eigen_seconds)
