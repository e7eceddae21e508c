"""Dev probe: moments exactness and PCA finiteness over the parity images, repeated builds."""
import os as _os, sys as _sys; _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1712_06326_b200 as zb
import workloads
g = np.load("tests/golden/reference_vectors.npz")
imgs = []
for tag in ("eval_64x64_g_s90_m91", "eval_48x40_c_s101_m102", "eval_60x50_c_s7_m8", "eval_96x80_g_s11_m12"):
    im = g[tag + "__image"]
    imgs.append((tag, im.squeeze(-1) if im.shape[-1] == 1 else im, g[tag + "__known"]))
for tag, img, kn in imgs:
    for rep in range(3):
        mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8))
        s, S = mi.moments()
        rs, rS = oracle.patch_moments(img, 9, mi.dictionary)
        ok = np.array_equal(s, rs) and np.array_equal(S, rS)
        bad = [l for l in range(8) if not np.isfinite(mi.layout(l)["components"]).all()]
        print(tag, rep, "moments ok" if ok else "MOMENTS DIFFER", "nan layouts", bad, "n", mi.n)
