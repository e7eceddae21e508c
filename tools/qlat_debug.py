"""Dev probe: compare the low-latency query (k_query_lat) with the oracle on the golden images."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, workloads
import paper_1712_06326_b200 as zb
from tests.helpers import fillfront, pca_of
g = np.load("tests/golden/reference_vectors.npz")
tag = "eval_64x64_g_s90_m91"
img, kn = g[tag + "__image"].squeeze(-1), g[tag + "__known"]
mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8))
pm, pc = pca_of(mi)
om = oracle.MultiIndex(img, kn, 9, 0.6, 8, pca_mean=pm, pca_comp=pc)
print("n", mi.n, "nblk", (mi.n + 255) // 256)
bad = 0
for i, (x, y) in enumerate(fillfront(kn)):
    if i % 5: continue
    tv, tk = oracle.extract_patch_clamped(img, kn, x, y, 9)
    for k in (8, 80):
        (key, cost, err, lid, ncand), cands = mi.query_best_patch(tv, tk, k, 0, return_candidates=True)
        best, rlid, rn, rknn = om.query_best_patch(img, tv, tk, k, 0)
        ok = np.array_equal(cands, rknn) and (cost << 32 | key) == best
        if not ok:
            bad += 1
            if bad < 4:
                print("MISMATCH k", k, "lid", lid, rlid, "n", ncand, rn, "best", (cost << 32 | key) == best)
                print(" got ", (cands[:12] >> 32).tolist(), (cands[-4:] >> 32).tolist())
                print(" want", (rknn[:12] >> 32).tolist(), (rknn[-4:] >> 32).tolist())
                print(" q", mi.make_query(lid, tv, tk).tolist())
print("bad", bad)
