"""dev probe: a few cfg2 fill-loop queries with ZI_DEBUG_QUERY output."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import numpy as np

import oracle
import paper_1712_06326_b200 as zb
import workloads
from tests.helpers import fillfront

img, kn, p = workloads.cfg2()
mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=11, dims=12, knn=80))
front = fillfront(kn)
for i in range(0, len(front), len(front) // 12):
    x, y = front[i]
    tv, tk = oracle.extract_patch_clamped(img, kn, x, y, 11)
    mi.query_best_patch(tv, tk)
