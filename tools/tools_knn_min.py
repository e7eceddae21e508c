"""dev repro: bare-index knn on the golden uniform_D4 vectors."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import numpy as np

import paper_1712_06326_b200 as zb

g = np.load("tests/golden/reference_vectors.npz")
coords = g["uniform_D4__coords"]
idx = zb.ZCurveIndex.from_descriptors(coords, np.arange(coords.shape[0], dtype=np.uint32), 4)
for qi, q in enumerate(g["uniform_D4__queries"]):
    for k in (1, 10, 80):
        r = idx.knn(q, k)
        ok = np.array_equal(r, g[f"uniform_D4__knn_l2_k{k}"][qi])
        print(qi, k, ok, flush=True)
