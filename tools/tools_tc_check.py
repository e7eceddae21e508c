"""Dev probe: repeat small builds and compare the tensor-core moments with the oracle each time."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import sys
import numpy as np
sys.path.insert(0, "tests")
import oracle
import paper_1712_06326_b200 as zb
import workloads
img, kn = workloads.small_image(70, 90, 3, seed=21, hole_frac=0.08)
bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8))
    s, S = mi.moments()
    rs, rS = oracle.patch_moments(img, 9, mi.dictionary)
    ok_s = np.array_equal(s, rs)
    ok_S = np.array_equal(S, rS)
    if not (ok_s and ok_S):
        bad += 1
        d = np.argwhere(S != rS)
        print(it, "sums ok" if ok_s else f"sums bad {np.sum(s != rs)}", "gram bad", len(d), d[:5].tolist(),
              (S - rS)[tuple(d[0])] if len(d) else "")
print("bad", bad)
