"""GPU parity: every sm_100a kernel, through the C ABI, against the CPU oracle / the reference's
own vectors.  Bit-exact for all integer, byte and index work; the PCA eigen-solve (fp64, the one
floating-point product whose order is not pinned) is checked by tolerance."""
import numpy as np
import pytest

import oracle
import workloads
from tests.helpers import fillfront, is_morton_sorted, pca_of

pytestmark = pytest.mark.gpu

L2, L1 = 0, 1


# ------------------------------------------------------------------ z-curve index vs the reference
@pytest.mark.parametrize("kind", ["uniform", "clustered"])
@pytest.mark.parametrize("D", [4, 8, 10, 16])
def test_from_descriptors_matches_reference_vectors(zb, golden, kind, D):
    tag = f"{kind}_D{D}"
    coords = golden[tag + "__coords"]
    keys = np.arange(coords.shape[0], dtype=np.uint32)
    idx = zb.ZCurveIndex.from_descriptors(coords, keys, D)
    c, k = idx.export()
    assert np.array_equal(c, golden[tag + "__sorted_coords"])
    assert np.array_equal(k, golden[tag + "__sorted_keys"])


@pytest.mark.parametrize("kind", ["uniform", "clustered"])
@pytest.mark.parametrize("D", [4, 8, 10, 16])
def test_knn_matches_reference_vectors(zb, golden, kind, D):
    tag = f"{kind}_D{D}"
    coords = golden[tag + "__coords"]
    idx = zb.ZCurveIndex.from_descriptors(coords, np.arange(coords.shape[0], dtype=np.uint32), D)
    for norm, nname in ((L2, "l2"), (L1, "l1")):
        for k in (1, 10, 80):
            ref = golden[f"{tag}__knn_{nname}_k{k}"]
            for qi, q in enumerate(golden[tag + "__queries"]):
                got = idx.knn(q, k, norm=norm)
                assert np.array_equal(got, ref[qi]), (norm, k, qi)


def test_from_descriptors_unsorted_keys(zb):
    rng = np.random.default_rng(3)
    n, D = 50000, 6
    coords = (rng.integers(0, 256, (n, D)) // 16 * 16).astype(np.uint8)  # many ties
    keys = rng.permutation(np.arange(n, dtype=np.uint32) * 7 + 3).astype(np.uint32)
    idx = zb.ZCurveIndex.from_descriptors(coords, keys, D)
    c, k = idx.export()
    rc, rk = oracle.from_descriptors(coords, keys)
    assert np.array_equal(c, rc) and np.array_equal(k, rk)


@pytest.mark.parametrize("D", [1, 3, 4, 7, 8, 12, 16, 20, 32])
def test_from_descriptors_all_widths(zb, D):
    rng = np.random.default_rng(D)
    n = 9000 + 37 * D
    coords = rng.integers(0, 256, (n, D)).astype(np.uint8)
    coords[::3] = coords[::3] // 64 * 64
    keys = np.arange(n, dtype=np.uint32)
    c, k = zb.ZCurveIndex.from_descriptors(coords, keys, D).export()
    rc, rk = oracle.from_descriptors(coords, keys)
    assert np.array_equal(c, rc) and np.array_equal(k, rk)


@pytest.mark.parametrize("D,kind", [(4, "clustered"), (8, "clustered"), (8, "uniform"), (12, "clustered"),
                                    (16, "uniform")])
@pytest.mark.parametrize("k", [1, 80, 160, 1000, 3000])
def test_knn_random_vs_linear_oracle(zb, D, kind, k):
    rng = np.random.default_rng(100 + D + k)
    n = 120000
    if kind == "uniform":
        coords = rng.integers(0, 256, (n, D)).astype(np.uint8)
    else:
        centers = rng.integers(0, 256, (12, D))
        lab = rng.integers(0, 12, n)
        coords = np.clip(np.rint(centers[lab] + rng.normal(0, 6, (n, D))), 0, 255).astype(np.uint8)
    keys = np.arange(n, dtype=np.uint32)
    idx = zb.ZCurveIndex.from_descriptors(coords, keys, D)
    sc, sk = idx.export()
    for t in range(4):
        q = coords[rng.integers(0, n)] if t % 2 == 0 else rng.integers(0, 256, D).astype(np.uint8)
        for norm in (L2, L1):
            got = idx.knn(q, k, norm=norm)
            ref = oracle.knn_linear(sc, sk, q, k, norm)
            assert np.array_equal(got, ref), (t, norm)


def test_knn_edge_cases(zb):
    rng = np.random.default_rng(9)
    coords = rng.integers(0, 256, (37, 5)).astype(np.uint8)
    keys = np.arange(37, dtype=np.uint32)
    idx = zb.ZCurveIndex.from_descriptors(coords, keys, 5)
    q = rng.integers(0, 256, 5).astype(np.uint8)
    for k in (0, 1, 36, 37, 38, 500):
        got = idx.knn(q, k)
        ref = oracle.knn_linear(coords, keys, q, k, L2)
        assert np.array_equal(got, ref), k
    # all-identical coordinates: pure key order
    same = np.full((1000, 4), 77, dtype=np.uint8)
    idx2 = zb.ZCurveIndex.from_descriptors(same, np.arange(1000, dtype=np.uint32), 4)
    got = idx2.knn(same[0], 80)
    assert np.array_equal(got & np.uint64(0xFFFFFFFF), np.arange(80, dtype=np.uint64))
    # single entry
    one = zb.ZCurveIndex.from_descriptors(coords[:1], keys[:1], 5)
    assert np.array_equal(one.knn(q, 10), oracle.knn_linear(coords[:1], keys[:1], q, 10, L2))


def test_knn_batch(zb):
    rng = np.random.default_rng(11)
    coords = rng.integers(0, 256, (20000, 8)).astype(np.uint8)
    keys = np.arange(20000, dtype=np.uint32)
    idx = zb.ZCurveIndex.from_descriptors(coords, keys, 8)
    sc, sk = idx.export()
    qs = rng.integers(0, 256, (16, 8)).astype(np.uint8)
    out, cnt = idx.knn_batch(qs, 40)
    for i in range(16):
        assert cnt[i] == 40
        assert np.array_equal(out[i], oracle.knn_linear(sc, sk, qs[i], 40, L2))


def test_binding_knn_search_matches_numpy(zb):
    """proj/tests/python/test_smoke.py:37-48 protocol against the mirror binding."""
    rng = np.random.default_rng(0)
    points = rng.integers(0, 256, size=(5000, 8)).astype(np.uint8)
    for norm in ("l2", "l1"):
        for k in (1, 15):
            query = rng.integers(0, 256, size=8).astype(np.uint8)
            dist, idx = zb.knn_search(points, query, k=k, norm=norm)
            diff = points.astype(np.int64) - query.astype(np.int64)
            ref = (diff ** 2).sum(axis=1) if norm == "l2" else np.abs(diff).sum(axis=1)
            order = np.lexsort((np.arange(len(points)), ref))[:k]
            assert np.array_equal(idx, order)
            assert np.array_equal(dist, ref[order])


# ------------------------------------------------------------------ index build
def _images(golden):
    out = []
    for tag, frac_tag in (("eval_64x64_g_s90_m91", True), ("eval_48x40_c_s101_m102", True),
                          ("eval_60x50_c_s7_m8", True), ("eval_96x80_g_s11_m12", True)):
        out.append((tag, golden[tag + "__image"].squeeze(-1) if golden[tag + "__image"].shape[-1] == 1
                    else golden[tag + "__image"], golden[tag + "__known"]))
    img, kn = workloads.small_image(70, 90, 3, seed=21, hole_frac=0.08)
    out.append(("small_rgb", img, kn))
    img, kn = workloads.small_image(64, 64, 1, seed=22, hole_frac=0.12)
    out.append(("small_gray", img, kn))
    return out


def test_dictionary_collect(zb, golden):
    for tag, img, kn in _images(golden):
        for K in (3, 5, 9, 11):
            mi_dict = oracle.collect_dictionary(kn, K)
            if mi_dict.size == 0:
                continue
            cfg = zb.index_config(patch_size=K, dims=4)
            mi = zb.MultiIndex(img, kn, cfg)
            assert np.array_equal(mi.dictionary, mi_dict), (tag, K)


@pytest.mark.parametrize("h,w", [(45, 64), (37, 132), (64, 68), (23, 24), (41, 63), (50, 130)])
def test_dictionary_collect_window_flag_shapes(zb, h, w):
    """The fused window-flag kernel (word-aligned rows: 4 columns x 8 rows per thread, K <= 9, or
    4 x 2 for K <= 17) and the two-kernel fallback (w % 4 != 0, larger K): heights that are not a
    multiple of the rows per thread, widths whose last word is partial, holes on the borders --
    the dictionary equals the oracle's."""
    img, kn = workloads.small_image(h, w, 1, seed=h * 131 + w, hole_frac=0.1)
    kn[0, :3] = 0
    kn[-1, -2:] = 0
    kn[h // 2, 0] = 0
    for K in (3, 5, 7, 9, 11, 13, 17, 19):
        if K > min(h, w):
            continue
        ref = oracle.collect_dictionary(kn, K)
        if ref.size == 0:
            continue
        mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=K, dims=2))
        assert np.array_equal(mi.dictionary, ref), (h, w, K)


def test_build_to_overlapped_copies_equal_build(zb, golden):
    """zi_multi_index_build_to (image upload and dictionary download on the copy stream beside the
    build) returns the dictionary and builds the same 8 indices as zi_multi_index_build."""
    import ctypes as C
    from paper_1712_06326_b200 import _lib
    L = _lib.lib()
    for tag, img, kn in _images(golden)[:3]:
        cfg = zb.index_config(patch_size=9, dims=6)
        ref = zb.MultiIndex(img, kn, cfg)
        h_, w_ = kn.shape
        ch = 1 if img.ndim == 2 else img.shape[2]
        cap = (w_ - 8) * (h_ - 8)
        keys = np.zeros(cap, np.uint32)
        n = C.c_uint64(0)
        hmi = C.c_void_p()
        _lib.check(L.zi_multi_index_build_to(ref.ctx.h, _lib.ptr(np.ascontiguousarray(img), _lib.u8p),
                                             _lib.ptr(np.ascontiguousarray(kn), _lib.u8p), w_, h_, ch, C.byref(cfg),
                                             _lib.ptr(keys, _lib.u32p), cap, C.byref(n), C.byref(hmi)))
        try:
            assert n.value == ref.n, tag
            assert np.array_equal(keys[:n.value], ref.dictionary), tag
            for l in range(8):
                c = np.zeros((ref.n, ref.dims), np.uint8)
                k = np.zeros(ref.n, np.uint32)
                _lib.check(L.zi_multi_index_layout_index(hmi, l, _lib.ptr(c, _lib.u8p), _lib.ptr(k, _lib.u32p)))
                rc, rk = ref.index_arrays(l)
                assert np.array_equal(c, rc) and np.array_equal(k, rk), (tag, l)
        finally:
            _lib.check(L.zi_multi_index_destroy(hmi))
        small = np.zeros(max(1, ref.n - 1), np.uint32)
        with pytest.raises(ValueError):  # ZI_E_INVALID: the dictionary does not fit
            _lib.check(L.zi_multi_index_build_to(ref.ctx.h, _lib.ptr(np.ascontiguousarray(img), _lib.u8p),
                                                 _lib.ptr(np.ascontiguousarray(kn), _lib.u8p), w_, h_, ch,
                                                 C.byref(cfg), _lib.ptr(small, _lib.u32p), small.size, C.byref(n),
                                                 C.byref(hmi)))


@pytest.mark.parametrize("K,ch,D", [(9, 1, 8), (9, 1, 4), (11, 3, 12), (9, 1, 16)])
def test_fused_lsd_build_equals_oracle(zb, K, ch, D):
    """The LSD sort policy: the sort's last pass writes the 8 indices (dim planes, keys carried as
    the record payload) and one kernel adds the bboxes -- byte-equal to the oracle's build_index."""
    from tests.helpers import pca_of
    img, kn = workloads.small_image(120, 104, ch, seed=40 + D, hole_frac=0.1)
    ctx = zb.Context.default()
    ctx.set_sort_policy(D, -1)
    try:
        ctx.set_profiling(True)
        mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=K, dims=D), ctx=ctx)
        prof = ctx.profile()
        ctx.set_profiling(False)
        assert mi.dims == D
        assert prof.get("index_bbox", (0.0, 0))[1] == 1, "the fused final pass did not run"
        assert prof.get("finalize_index", (0.0, 0))[1] == 0
        pm, pc = pca_of(mi)
        om = oracle.MultiIndex(img, kn, K, 0.6, D, pca_mean=pm, pca_comp=pc)
        for l in range(8):
            c, k = mi.index_arrays(l)
            ref = om.index(l)
            assert np.array_equal(c, ref.coords) and np.array_equal(k, ref.keys), (D, l)
            lay = mi.layout(l)
            assert np.array_equal(lay["lo"], ref.lo) and np.array_equal(lay["hi"], ref.hi), (D, l)
        # the bboxes the queries prune with: a query equals the oracle's
        ys, xs = np.nonzero(kn == 0)
        tv, tk = oracle.extract_patch_clamped(img, kn, int(xs[0]), int(ys[0]) - 1, K)
        got = mi.query_best_patch(tv, tk)
        best, lid, ncand, _ = om.query_best_patch(img, tv, tk, 80)
        assert (got[1] << 32 | got[0]) == best and got[3] == lid and got[4] == ncand, D
    finally:
        ctx.set_profiling(False)
        ctx.set_sort_policy(D, 0)


def test_empty_dictionary_raises(zb):
    img = np.zeros((20, 20), np.uint8)
    with pytest.raises(zb.EmptyDictionaryError):
        zb.MultiIndex(img, np.zeros((20, 20), np.uint8), zb.index_config(dims=4))


def test_moments_exact(zb, golden):
    for tag, img, kn in _images(golden)[:3]:
        mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=6))
        s, S = mi.moments()
        rs, rS = oracle.patch_moments(img, 9, mi.dictionary)
        assert np.array_equal(s, rs) and np.array_equal(S, rS), tag


def _check_pca(mi, K, ch, tag):
    s, S = mi.moments()
    for l in range(8):
        lay = mi.layout(l)
        cols = oracle.layout_columns(lay["pixels"], K, ch)
        mean, cov = oracle.layout_covariance(s, S, mi.n, cols)
        assert np.array_equal(lay["mean"], mean), (tag, l)
        comp, eig = oracle.pca_from_cov(cov, mi.dims)
        np.testing.assert_allclose(lay["eigenvalues"], eig, rtol=1e-9, atol=1e-9 * eig[0])
        # orthonormal, eigen-residual small, and equal to the oracle's where the spectrum is simple
        C = lay["components"]
        np.testing.assert_allclose(C @ C.T, np.eye(mi.dims), atol=1e-10)
        res = cov @ C.T - C.T * lay["eigenvalues"]
        assert np.abs(res).max() <= 1e-9 * max(1.0, eig[0]), (tag, l)
        gaps = np.abs(np.diff(eig))
        for d in range(mi.dims):
            g = min(gaps[d - 1] if d > 0 else np.inf, gaps[d] if d < len(gaps) else np.inf)
            if g > 1e-6 * eig[0]:
                np.testing.assert_allclose(C[d], comp[d], atol=1e-7)
            # reference sign rule: the first largest-magnitude entry is positive
            i = int(np.argmax(np.abs(C[d])))
            assert C[d][i] > 0, (tag, l, d)


def test_pca_matches_oracle_fit(zb, golden):
    for tag, img, kn in _images(golden)[:4]:
        mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8))
        assert mi.info.pca_on_device == 1
        _check_pca(mi, 9, 1 if img.ndim == 2 else img.shape[2], tag)


@pytest.mark.parametrize("K,dims,device", [(11, 12, 1), (11, 32, 1), (13, 12, 0), (3, 9, 1)])
def test_pca_rgb_device_and_host_paths(zb, K, dims, device):
    """mc = m*C: K=11 RGB -> 219 (device k_pca), K=13 RGB -> 303 (host fallback)."""
    img, kn = workloads.small_image(80, 72, 3, seed=K + dims, hole_frac=0.1)
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=K, dims=dims))
    assert mi.info.pca_on_device == device
    _check_pca(mi, K, 3, (K, dims))


def test_pca_constant_image(zb):
    """Zero covariance: eigenvalues 0, components still orthonormal, build still bit-exact."""
    img = np.full((30, 30), 77, np.uint8)
    mi = zb.MultiIndex(img, np.ones((30, 30), np.uint8), zb.index_config(patch_size=5, dims=4))
    for l in range(8):
        lay = mi.layout(l)
        assert (lay["eigenvalues"] == 0).all()
        C = lay["components"]
        np.testing.assert_allclose(C @ C.T, np.eye(mi.dims), atol=1e-10)
        c, _ = mi.index_arrays(l)
        assert (c == 0).all()


def test_build_bitexact_against_oracle(zb, golden):
    for tag, img, kn in _images(golden):
        for dims in (4, 8):
            mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=dims))
            pm, pc = pca_of(mi)
            om = oracle.MultiIndex(img, kn, 9, 0.6, dims, pca_mean=pm, pca_comp=pc)
            for l in range(8):
                c, k = mi.index_arrays(l)
                ref = om.index(l)
                lay = mi.layout(l)
                assert np.array_equal(lay["lo"], ref.lo) and np.array_equal(lay["hi"], ref.hi), (tag, l)
                assert np.array_equal(c, ref.coords) and np.array_equal(k, ref.keys), (tag, l)


def test_build_tiny_dictionary_shrinks_dims(zb, golden):
    """A1: D = min(cfg.dims, m*C, n) -- one-patch dictionary gives D = 1 (test_builder.cpp:41-50)."""
    img = golden["eval_20x20_g_s1__image"][:9, :9, 0].copy()
    mi = zb.MultiIndex(img, np.ones((9, 9), np.uint8), zb.index_config(patch_size=9, dims=4))
    assert mi.n == 1 and mi.dims == 1


def test_constant_image_ties_in_key_order(zb):
    """test_builder.cpp:52-63: identical content -> row-major key order."""
    img = np.full((12, 24), 120, np.uint8)
    mi = zb.MultiIndex(img, np.ones((12, 24), np.uint8), zb.index_config(patch_size=9, dims=2))
    for l in range(8):
        _, k = mi.index_arrays(l)
        assert (np.diff(k.astype(np.int64)) > 0).all()


def test_rebuild_bit_identical(zb, golden):
    img = golden["eval_32x24_c_s4__image"]
    kn = np.ones(img.shape[:2], np.uint8)
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9))
    a = [mi.index_arrays(l) for l in range(8)]
    la = [mi.layout(l) for l in range(8)]
    mi.rebuild()
    for l in range(8):
        c, k = mi.index_arrays(l)
        assert np.array_equal(c, a[l][0]) and np.array_equal(k, a[l][1])
        for f in ("mean", "components", "lo", "hi"):
            assert np.array_equal(mi.layout(l)[f], la[l][f])


# ------------------------------------------------------------------ queries
def _query_cases(img, kn, stride=3):
    out = []
    for i, (x, y) in enumerate(fillfront(kn)):
        if i % stride == 0:
            out.append(oracle.extract_patch_clamped(img, kn, x, y, 9))
    return out


@pytest.mark.parametrize("k", [1, 8, 80, 300])
@pytest.mark.parametrize("norm", [L2, L1])
def test_query_best_patch_matches_oracle(zb, golden, k, norm):
    for tag, img, kn in _images(golden)[:4]:
        mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8, norm=norm))
        pm, pc = pca_of(mi)
        om = oracle.MultiIndex(img, kn, 9, 0.6, 8, pca_mean=pm, pca_comp=pc)
        for tv, tk in _query_cases(img, kn, 5):
            (key, cost, err, lid, ncand), cands = mi.query_best_patch(tv, tk, k, norm, return_candidates=True)
            best, rlid, rn, rknn = om.query_best_patch(img, tv, tk, k, norm)
            assert lid == rlid and ncand == rn, tag
            assert np.array_equal(cands, rknn), tag
            assert (cost << 32 | key) == best, tag


def test_query_with_k_equal_n_is_brute_force(zb, golden):
    """test_engine.cpp:210-231: k = dictionary size -> filter+refine == brute force."""
    img = golden["eval_40x32_g_s84__image"][:, :, 0]
    kn = np.ones(img.shape, np.uint8)
    kn[10:18, 22:30] = 0
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8))
    n = mi.n
    for tv, tk in _query_cases(img, kn, 3):
        key, cost, *_ = mi.query_best_patch(tv, tk, n)
        bkey, bcost, _ = mi.brute_force_best(tv, tk)
        assert key == bkey and cost == bcost


@pytest.mark.parametrize("norm", [L2, L1])
def test_brute_force_matches_oracle(zb, golden, norm):
    for tag, img, kn in _images(golden):
        mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=4))
        d = mi.dictionary
        for tv, tk in _query_cases(img, kn, 9):
            key, cost, _ = mi.brute_force_best(tv, tk, norm)
            assert (cost << 32 | key) == oracle.brute_force_best(img, tv, tk, 9, d, norm), tag


def test_brute_force_exact_match_cost_zero(zb, golden):
    """test_engine.cpp:258-270"""
    img = golden["eval_30x30_g_s91__image"][:, :, 0]
    kn = np.ones((30, 30), np.uint8)
    kn[20:29, 20:29] = 0
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=4))
    full = np.ones((30, 30), np.uint8)
    tv, tk = oracle.extract_patch_clamped(img, full, 6, 6, 9)
    key, cost, _ = mi.brute_force_best(tv, tk)
    assert cost == 0 and key == (2 << 16 | 2)


# ------------------------------------------------------------------ fill loop end to end
def _compare_runs(out, recs, rout, rrecs):
    assert len(recs) == len(rrecs)
    assert np.array_equal(recs["target_x"], rrecs["tx"]) and np.array_equal(recs["target_y"], rrecs["ty"])
    assert np.array_equal(recs["source_key"], (rrecs["sy"].astype(np.uint32) << 16) | rrecs["sx"].astype(np.uint32))
    assert np.array_equal(recs["cost"], rrecs["cost"])
    assert np.array_equal(out, rout)


@pytest.mark.parametrize("case", range(4))
def test_inpaint_bitexact_against_oracle(zb, golden, case):
    tag, img, kn = _images(golden)[case]
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8, knn=12))
    pm, pc = pca_of(mi)
    out, recs, stats = mi.inpaint(oracle=True, oracle_stride=2)
    rout, rrecs = oracle.inpaint(img, kn, 9, 0.6, 8, knn=12, oracle=True, oracle_stride=2, pca_mean=pm, pca_comp=pc)
    _compare_runs(out, recs, rout, rrecs)
    assert np.array_equal(recs["layout_id"], rrecs["layout_id"])
    bf = recs["bf_error"]
    rbf = rrecs["bf_error"]
    assert np.array_equal(np.isnan(bf), np.isnan(rbf))
    assert np.array_equal(bf[~np.isnan(bf)], rbf[~np.isnan(rbf)])
    known = kn != 0
    assert np.array_equal(out[known], img[known])  # conservation


def test_inpaint_brute_force_mode(zb, golden):
    tag, img, kn = _images(golden)[1]
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8))
    out, recs, _ = mi.inpaint(brute_force=True)
    rout, rrecs = oracle.inpaint(img, kn, 9, 0.6, 8, brute_force=True)
    _compare_runs(out, recs, rout, rrecs)


def test_binding_inpaint_roundtrip(zb):
    """proj/tests/python/test_smoke.py:51-63 + 65-75 protocols on the mirror binding."""
    rng = np.random.default_rng(3)
    yy, xx = np.mgrid[0:60, 0:80]
    base = 120 + 60 * np.sin(0.21 * xx + 0.13 * yy) + 0.2 * xx
    img = np.stack([base + 10 * c for c in range(3)], axis=-1) + rng.integers(-6, 7, size=(60, 80, 3))
    img = np.clip(img, 0, 255).astype(np.uint8)
    mask = np.full((60, 80), 255, dtype=np.uint8)
    mask[20:24, 10:70] = 0
    mask[40:43, 5:60] = 0
    out = zb.inpaint(img, mask, dims=6, knn=8, workers=2)
    assert out["image"].shape == img.shape
    known = mask >= 128
    assert np.array_equal(out["image"][known], img[known])
    assert out["stats"]["iterations"] == len(out["records"]) > 0
    g = img[:40, :50, 0].copy()
    m2 = np.full((40, 50), 255, dtype=np.uint8)
    m2[15:18, 8:40] = 0
    o2 = zb.inpaint(g, m2, dims=6, knn=6, workers=1, oracle=True)
    assert o2["stats"]["mean_ae"] is not None and o2["stats"]["mean_ae"] >= 0.0
    for rec in o2["records"]:
        assert rec["bf_error"] is not None and rec["z_error"] >= rec["bf_error"] - 1e-12
    with pytest.raises(Exception):
        zb.inpaint(img, np.zeros((10, 10), dtype=np.uint8))
    with pytest.raises(Exception):
        zb.inpaint(img, np.zeros((60, 80), dtype=np.uint8))


def test_inpaint_degenerate_masks(zb, golden):
    """test_engine.cpp:337-353"""
    img = golden["eval_20x20_g_s1__image"][:, :, 0]
    cfg = zb.index_config(patch_size=9, dims=4)
    out, recs, _ = zb.inpaint_raw(img, np.ones((20, 20), np.uint8), cfg)
    assert len(recs) == 0 and np.array_equal(out, img)
    one = np.ones((20, 20), np.uint8)
    one[10, 10] = 0
    out, recs, st = zb.inpaint_raw(img, one, cfg)
    assert len(recs) == 1 and st.iterations == 1


@pytest.mark.slow
def test_cfg1_end_to_end_bitexact(zb):
    img, kn, p = workloads.cfg1()
    cfg = zb.index_config(patch_size=9, dims=8, knn=80)
    mi = zb.MultiIndex(img, kn, cfg)
    assert mi.n == int(oracle.collect_dictionary(kn, 9).size) == 58368
    pm, pc = pca_of(mi)
    om = oracle.MultiIndex(img, kn, 9, 0.6, 8, pca_mean=pm, pca_comp=pc)
    for l in range(8):
        c, k = mi.index_arrays(l)
        r = om.index(l)
        assert np.array_equal(c, r.coords) and np.array_equal(k, r.keys)
    out, recs, _ = mi.inpaint()
    rout, rrecs = oracle.inpaint(img, kn, 9, 0.6, 8, knn=80, mi=om)
    _compare_runs(out, recs, rout, rrecs)


@pytest.mark.slow
def test_cfg2_build_properties(zb):
    """Full-size cfg2 build: permutation, Morton sortedness, lo/hi, and spot knn vs the oracle."""
    img, kn, p = workloads.cfg2()
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=11, dims=12))
    d = mi.dictionary
    assert np.array_equal(d, oracle.collect_dictionary(kn, 11))
    rng = np.random.default_rng(0)
    for l in (0, 5):
        c, k = mi.index_arrays(l)
        assert np.array_equal(np.sort(k), d)
        assert is_morton_sorted(c, k)
        lay = mi.layout(l)
        sub = rng.choice(len(d), 2000, replace=False)
        lo, hi, coords, y = oracle.project_build(img, d[sub], lay["pixels"], lay["mean"], lay["components"])
        assert (y.min(0) >= lay["lo"]).all() and (y.max(0) <= lay["hi"]).all()
        pos = np.searchsorted(d, d[sub])
        # quantised bytes of the sampled patches equal the oracle quantiser with the global lo/hi
        order = np.argsort(k)
        q = np.array([[oracle.quantize(lay["lo"][j], lay["hi"][j], y[i, j]) for j in range(mi.dims)] for i in range(200)])
        assert np.array_equal(c[order[pos[:200]]], q)
        idx = mi.index(l)
        for t in range(3):
            qv = c[rng.integers(0, len(k))]
            assert np.array_equal(idx.knn(qv, 80), oracle.knn_linear(c, k, qv, 80))


@pytest.mark.slow
def test_cfg4_build_properties(zb):
    """cfg4 (4096^2 gray, K=9, D=8, n ~ 15M): permutation, Morton order with key tie-break,
    lo/hi bound the projections, sampled quantised bytes equal the oracle's, spot knn."""
    img, kn, p = workloads.cfg4()
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8))
    d = mi.dictionary
    assert np.array_equal(d, oracle.collect_dictionary(kn, 9))
    rng = np.random.default_rng(4)
    for l in (0, 3, 7):
        c, k = mi.index_arrays(l)
        assert np.array_equal(np.sort(k), d)
        assert is_morton_sorted(c, k)
        lay = mi.layout(l)
        sub = rng.choice(len(d), 2000, replace=False)
        lo, hi, coords, y = oracle.project_build(img, d[sub], lay["pixels"], lay["mean"], lay["components"])
        assert (y.min(0) >= lay["lo"]).all() and (y.max(0) <= lay["hi"]).all()
        pos = np.searchsorted(d, d[sub])
        order = np.argsort(k)
        q = np.array([[oracle.quantize(lay["lo"][j], lay["hi"][j], y[i, j]) for j in range(mi.dims)] for i in range(200)])
        assert np.array_equal(c[order[pos[:200]]], q)
        idx = mi.index(l)
        for t in range(2):
            qv = c[rng.integers(0, len(k))]
            assert np.array_equal(idx.knn(qv, 80), oracle.knn_linear(c, k, qv, 80))


@pytest.mark.parametrize("D", [4, 8, 16])
def test_knn_batch_cfg5_like_vs_oracle(zb, D):
    coords, queries = workloads.cfg5_descriptors(60000, D, 64, seed=D)
    keys = np.arange(coords.shape[0], dtype=np.uint32)
    idx = zb.ZCurveIndex.from_descriptors(coords, keys, D)
    sc, sk = idx.export()
    for k in (1, 80, 256):
        out, cnt = idx.knn_batch(queries, k)
        ms, stats, (o2, c2) = idx.knn_batch_bench(queries, k, reps=1, return_results=True)
        assert np.array_equal(out, o2) and np.array_equal(cnt, c2)
        for i in range(0, 64, 7):
            ref = oracle.knn_linear(sc, sk, queries[i], k)
            assert cnt[i] == ref.size and np.array_equal(out[i, :cnt[i]], ref), (k, i)


# ------------------------------------------------------------------ ZIDX1 persistence
def _parse_zidx1(path, K, C):
    """Restated reader of the reference's format (proj/include/zinpaint/io_index.hpp:10-17)."""
    import struct
    raw = open(path, "rb").read()
    off, blocks = 0, []
    for _ in range(8):
        assert raw[off:off + 5] == b"ZIDX1"
        off += 5
        k, cov, D, lid, n, ch = struct.unpack_from("<IdIIQI", raw, off)
        off += struct.calcsize("<IdIIQI")
        m = oracle.subset_layouts(k, cov)[0].shape[0] * ch
        f = lambda cnt: np.frombuffer(raw, np.float64, cnt, off)
        mean = f(m); off += 8 * m
        comp = f(D * m).reshape(D, m); off += 8 * D * m
        eig = f(D); off += 8 * D
        lo = f(D); off += 8 * D
        hi = f(D); off += 8 * D
        ent = np.frombuffer(raw, np.uint8, n * (D + 8), off).reshape(n, D + 8); off += n * (D + 8)
        coords = ent[:, :D].copy()
        xy = ent[:, D:].copy().view(np.uint32)
        keys = (xy[:, 1] << 16) | xy[:, 0]
        blocks.append(dict(K=k, coverage=cov, D=D, layout=lid, n=n, C=ch, mean=mean, comp=comp, eig=eig, lo=lo,
                           hi=hi, coords=coords, keys=keys))
    assert off == len(raw)
    return blocks


def test_zidx1_save_format_and_load_roundtrip(zb, golden, tmp_path):
    tag = "eval_48x40_c_s101_m102"
    img, kn = golden[tag + "__image"], golden[tag + "__known"]
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8))
    path = tmp_path / "idx.zidx"
    mi.save(path)
    blocks = _parse_zidx1(path, 9, 3)
    for l, b in enumerate(blocks):
        lay = mi.layout(l)
        c, k = mi.index_arrays(l)
        assert (b["K"], b["D"], b["layout"], b["n"], b["C"]) == (9, mi.dims, l, mi.n, 3)
        assert b["coverage"] == 0.6
        for f in ("mean", "eig", "lo", "hi"):
            np.testing.assert_array_equal(b[f], lay["eigenvalues" if f == "eig" else f])
        np.testing.assert_array_equal(b["comp"], lay["components"])
        assert np.array_equal(b["coords"], c) and np.array_equal(b["keys"], k)
    # load: same indices, models and query answers; the loaded object can run the fill loop
    ml = zb.MultiIndex.load(path, img, known=kn)
    assert ml.info.loaded == 1 and ml.n == mi.n and ml.dims == mi.dims
    assert np.array_equal(ml.dictionary, mi.dictionary)
    for l in range(8):
        for f in ("mean", "components", "eigenvalues", "lo", "hi"):
            assert np.array_equal(ml.layout(l)[f], mi.layout(l)[f])
        a, b = mi.index_arrays(l), ml.index_arrays(l)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for tv, tk in _query_cases(img, kn, stride=7):
        assert mi.query_best_patch(tv, tk) == ml.query_best_patch(tv, tk)
    o1, r1, _ = mi.inpaint()
    o2, r2, _ = ml.inpaint()
    assert np.array_equal(o1, o2) and np.array_equal(r1["source_key"], r2["source_key"])


def test_zidx1_load_resorts_and_rejects_bad_files(zb, golden, tmp_path):
    import struct
    tag = "eval_64x64_g_s90_m91"
    img, kn = golden[tag + "__image"].squeeze(-1), golden[tag + "__known"]
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=6))
    path = tmp_path / "a.zidx"
    mi.save(path)
    raw = bytearray(open(path, "rb").read())
    # shuffle the entries of block 0: load re-sorts (io_index.cpp:120)
    hdr = 5 + struct.calcsize("<IdIIQI")
    k, cov, D, lid, n, ch = struct.unpack_from("<IdIIQI", raw, 5)
    m = oracle.subset_layouts(k, cov)[0].shape[0] * ch
    e0 = hdr + 8 * (m + D * m + 3 * D)
    ent = np.frombuffer(bytes(raw[e0:e0 + n * (D + 8)]), np.uint8).reshape(n, D + 8)
    perm = np.random.default_rng(0).permutation(n)
    raw[e0:e0 + n * (D + 8)] = ent[perm].tobytes()
    shuffled = tmp_path / "s.zidx"
    open(shuffled, "wb").write(bytes(raw))
    ml = zb.MultiIndex.load(shuffled, img)
    a, b = mi.index_arrays(0), ml.index_arrays(0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # bad magic, truncation, bad header -> runtime errors (std::runtime_error in the reference)
    bad = tmp_path / "b.zidx"
    open(bad, "wb").write(b"ZIDX2" + bytes(raw[5:]))
    with pytest.raises(zb.ZIError):
        zb.MultiIndex.load(bad, img)
    open(bad, "wb").write(bytes(raw[: len(raw) - 7]))
    with pytest.raises(zb.ZIError):
        zb.MultiIndex.load(bad, img)
    hb = bytearray(raw)
    struct.pack_into("<I", hb, 5 + 4 + 8 + 4, 9)  # layout id 9
    open(bad, "wb").write(bytes(hb))
    with pytest.raises(zb.ZIError):
        zb.MultiIndex.load(bad, img)


# ------------------------------------------------------------------ cfg5 vector index
@pytest.mark.parametrize("n,dim,D", [(40000, 125, 8), (5000, 13, 16), (33000, 125, 16)])
def test_vector_index_vs_oracle(zb, n, dim, D):
    """Mean / covariance bit-exact in the canonical stripe order (FP64 MMA chains == sequential
    fma); PCA by tolerance; projection, quantiser, sort, make_query and k-NN bit-exact with the
    device PCA injected into the oracle."""
    X = workloads.cfg5_points(n, dims_in=dim, seed=n + dim)
    vi = zb.VectorIndex(X, D)
    assert vi.dims == min(D, dim, n)
    mod = vi.model()
    mean, cov = oracle.vec_mean_cov(X)
    assert np.array_equal(mod["mean"], mean)
    comp, eig = oracle.pca_from_cov(cov, vi.dims)
    np.testing.assert_allclose(mod["eigenvalues"], eig, rtol=1e-9, atol=1e-9 * eig[0])
    Cm = mod["components"]
    np.testing.assert_allclose(Cm @ Cm.T, np.eye(vi.dims), atol=1e-10)
    res = cov @ Cm.T - Cm.T * mod["eigenvalues"]
    assert np.abs(res).max() <= 1e-9 * max(1.0, eig[0])
    lo, hi, coords = oracle.vec_project(X, mod["mean"], Cm)
    assert np.array_equal(lo, mod["lo"]) and np.array_equal(hi, mod["hi"])
    rows = np.arange(n, dtype=np.uint32)
    rc, rk = oracle.from_descriptors(coords, rows)
    c, k = vi.index().export()
    assert np.array_equal(c, rc) and np.array_equal(k, rk)
    rng = np.random.default_rng(7)
    Q = workloads.cfg5_points(32, dims_in=dim, seed=99)
    known = (rng.random(Q.shape) >= 0.4).astype(np.uint8)
    qd = vi.make_queries(Q, known)
    for i in range(Q.shape[0]):
        assert np.array_equal(qd[i], oracle.vec_make_query(Q[i], known[i], mod["mean"], Cm, lo, hi))
    out, cnt = vi.knn(Q, known, k=80)
    for i in range(0, 32, 5):
        ref = oracle.knn_linear(rc, rk, qd[i], 80)
        assert cnt[i] == ref.size and np.array_equal(out[i, :cnt[i]], ref)


@pytest.mark.gpu
def test_build_deterministic_repeats(zb):
    """Window sort / tensor-core moments: repeated builds of one image are byte-identical
    (shared-memory or TMEM races show up as run-to-run differences)."""
    img, kn = workloads.small_image(70, 90, 3, seed=21, hole_frac=0.08)
    ref = None
    for _ in range(12):
        mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=8))
        got = [mi.index_arrays(l) for l in range(8)] + [mi.moments()]
        if ref is None:
            ref = got
            continue
        for a, b in zip(ref, got):
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ------------------------------------------------------------------ range-partitioned shards (§8(e))
def _sharded(zb, img, known, cfg, world, samples=64):
    from paper_1712_06326_b200 import sharding
    shards = [sharding.DeviceShard(img, known, cfg, r, world) for r in range(world)]
    info = sharding.build_sharded(shards, sharding.LoopbackComm(world), samples=samples)
    return sharding, shards, info


@pytest.mark.parametrize("world,channels,dims,samples", [(1, 1, 8, 64), (2, 1, 8, 64), (3, 3, 12, 16),
                                                         (4, 1, 4, 4), (5, 3, 8, 256)])
def test_sharded_build_equals_single_gpu_build(zb, world, channels, dims, samples):
    """Rank r's layout-l shard == positions shard_ranges(n, G)[r] of the single-GPU layout-l index
    (coords, keys), with the same PCA models and quantiser ranges on every rank."""
    img, known = workloads.small_image(72, 88, channels, seed=11 + world, hole_frac=0.08)
    cfg = zb.index_config(patch_size=9 if channels == 1 else 7, dims=dims, knn=24)
    mi = zb.MultiIndex(img, known, cfg)
    sharding, shards, info = _sharded(zb, img, known, cfg, world, samples)
    ranges = sharding.shard_ranges(mi.n, world)
    for r, sh in enumerate(shards):
        assert (sh.row_begin, sh.row_end) == ranges[r]
        assert sh.multi_index.n == ranges[r][1] - ranges[r][0]
        assert np.array_equal(sh.multi_index.dictionary, mi.dictionary[ranges[r][0]:ranges[r][1]])
    for l in range(8):
        c, k = mi.index_arrays(l)
        ref = mi.layout(l)
        for r, sh in enumerate(shards):
            b, e = ranges[r]
            cs, ks = sh.multi_index.index_arrays(l)
            assert np.array_equal(cs, c[b:e]) and np.array_equal(ks, k[b:e]), (l, r)
            lay = sh.multi_index.layout(l)
            for f in ("mean", "components", "eigenvalues", "lo", "hi"):
                assert np.array_equal(lay[f].view(np.uint64), ref[f].view(np.uint64)), (l, r, f)
    if world > 1:
        assert info["records_exchanged"] > 0


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_query_and_brute_force_equal_single_gpu(zb, world):
    """Merged per-shard k-NN + one refine == query_best_patch on the whole index; packed-min of
    the per-slice scans == brute_force_best (winner key and cost, every target)."""
    img, known = workloads.small_image(80, 96, 3, seed=21, hole_frac=0.1)
    cfg = zb.index_config(patch_size=7, dims=8, knn=32)
    mi = zb.MultiIndex(img, known, cfg)
    sharding, shards, _ = _sharded(zb, img, known, cfg, world)
    comm = sharding.LoopbackComm(world)
    targets = fillfront(known)[:12]
    assert len(targets) > 0
    for (x, y) in targets:
        tv, tk = oracle.extract_patch_clamped(img, known, int(x), int(y), 7)
        for k in (1, 32, 200):
            want = mi.query_best_patch(tv, tk, k)
            got = sharding.sharded_query(shards, comm, tv, tk, k, 0)
            for g in got:
                assert (g[0], g[1], g[3], g[4]) == (want[0], want[1], want[3], want[4]), (x, y, k)
        bw = mi.brute_force_best(tv, tk)
        for g in sharding.sharded_brute_force(shards, comm, tv, tk, 0):
            assert g == (bw[0], bw[1])


def test_sharded_build_cfg1(zb):
    """cfg1 (256^2 gray, 48^2 hole, K=9, D=8) over 4 shards == the single-GPU build."""
    img, known, _ = workloads.cfg1()
    cfg = zb.index_config(patch_size=9, dims=8, knn=80)
    mi = zb.MultiIndex(img, known, cfg)
    sharding, shards, info = _sharded(zb, img, known, cfg, 4, samples=256)
    for l in range(8):
        c, k = mi.index_arrays(l)
        cs = np.concatenate([sh.multi_index.index_arrays(l)[0] for sh in shards])
        ks = np.concatenate([sh.multi_index.index_arrays(l)[1] for sh in shards])
        assert np.array_equal(cs, c) and np.array_equal(ks, k), l
    # the rebalancing exchange only moves the sample-sort imbalance
    assert info["records_rebalanced"] < info["records_exchanged"]


def test_sharded_multi_index_over_nccl_world1(zb):
    """The torch.distributed path (NCCL, device tensors from the shard's own buffers) end to end
    at world size 1: ShardedMultiIndex == MultiIndex, queries included."""
    import torch
    import torch.distributed as dist

    from paper_1712_06326_b200 import sharding
    from tests.test_cpu import _free_port
    img, known = workloads.small_image(64, 72, 3, seed=31, hole_frac=0.1)
    cfg = zb.index_config(patch_size=7, dims=8, knn=16)
    mi = zb.MultiIndex(img, known, cfg)
    store = dist.TCPStore("127.0.0.1", _free_port(), 1, True)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1)
    try:
        smi = sharding.ShardedMultiIndex(img, known, cfg)
        for l in range(8):
            a, b = smi.index_arrays(l), mi.index_arrays(l)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        for (x, y) in fillfront(known)[:6]:
            tv, tk = oracle.extract_patch_clamped(img, known, int(x), int(y), 7)
            got, want = smi.query_best_patch(tv, tk), mi.query_best_patch(tv, tk)
            assert (got[0], got[1], got[3], got[4]) == (want[0], want[1], want[3], want[4])
            assert smi.brute_force_best(tv, tk) == mi.brute_force_best(tv, tk)[:2]
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ tensor-core projection filter
_FP64_DUMP = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1712_06326_b200 as zb, workloads
img, kn, p = getattr(workloads, sys.argv[2])()
mi = zb.MultiIndex(img, kn, zb.index_config(**p))
out = {}
for l in range(8):
    c, k = mi.index_arrays(l); lay = mi.layout(l)
    out[f"c{l}"], out[f"k{l}"], out[f"lo{l}"], out[f"hi{l}"] = c, k, lay["lo"], lay["hi"]
np.savez(sys.argv[3], **out)
"""


@pytest.mark.parametrize("D", [7, 8, 9, 10])
def test_projection_two_half_launch_vs_oracle(zb, D):
    """D = 7..10: both groups of four layouts in one projection launch (every A tile gathered once,
    two accumulator halves; the min / max pass keeps lane-slot extremes behind 32-bit filters) --
    all 8 indices and quantiser ranges byte-equal to the oracle fed the build's PCA model, on an
    image whose last tile is partial and whose rows break at holes."""
    from tests.helpers import pca_of
    img, kn = workloads.small_image(150, 131, 1, seed=70 + D, hole_frac=0.08)
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=9, dims=D))
    assert mi.dims == D and mi.n % 128 != 0
    pm, pc = pca_of(mi)
    om = oracle.MultiIndex(img, kn, 9, 0.6, D, pca_mean=pm, pca_comp=pc)
    for l in range(8):
        c, k = mi.index_arrays(l)
        ref = om.index(l)
        lay = mi.layout(l)
        assert np.array_equal(lay["lo"], ref.lo) and np.array_equal(lay["hi"], ref.hi), (D, l)
        assert np.array_equal(c, ref.coords) and np.array_equal(k, ref.keys), (D, l)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_projection_tc_equals_fp64_path(zb, cfg, tmp_path):
    """The int8 tensor-core filter + fix-up writes the same index bytes and quantiser ranges as the
    canonical FP64-MMA path (ZI_PROJ_FP64=1, another process) at full config size."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    dump = tmp_path / "fp64.npz"
    env = dict(os.environ, ZI_PROJ_FP64="1")
    subprocess.run([sys.executable, "-c", _FP64_DUMP, root, cfg, str(dump)], env=env, check=True, timeout=600)
    ref = np.load(dump)
    img, kn, p = getattr(workloads, cfg)()
    mi = zb.MultiIndex(img, kn, zb.index_config(**p))
    for l in range(8):
        c, k = mi.index_arrays(l)
        lay = mi.layout(l)
        assert np.array_equal(lay["lo"].view(np.uint64), ref[f"lo{l}"].view(np.uint64)), l
        assert np.array_equal(lay["hi"].view(np.uint64), ref[f"hi{l}"].view(np.uint64)), l
        assert np.array_equal(c, ref[f"c{l}"]) and np.array_equal(k, ref[f"k{l}"]), l


@pytest.mark.parametrize("case", ["two_level", "rgb_k7_d16", "rgb_k5_d1", "gray_k9_d13", "stripes_k11_rgb"])
def test_projection_tc_edge_cases_vs_oracle(zb, case):
    """Degenerate ranges (every pair re-projected exactly), the generic table gather (K*C not
    specialised), D = 1 and D = 16, ties at the extremes -- byte-equal to the oracle fed the
    build's PCA model."""
    rng = np.random.default_rng(17)
    if case == "two_level":
        img = (rng.random((40, 52)) < 0.5).astype(np.uint8) * 200 + 20
        K, D, C = 5, 4, 1
    elif case == "rgb_k7_d16":
        img, _ = workloads.small_image(56, 64, 3, seed=3, hole_frac=0.0)
        K, D, C = 7, 16, 3
    elif case == "rgb_k5_d1":
        img, _ = workloads.small_image(40, 48, 3, seed=4, hole_frac=0.0)
        K, D, C = 5, 1, 3
    elif case == "gray_k9_d13":
        img, _ = workloads.small_image(64, 72, 1, seed=5, hole_frac=0.0)
        K, D, C = 9, 13, 1
    else:  # vertical stripes: most components see a handful of distinct values
        x = np.arange(60)[None, :, None]
        img = np.broadcast_to(((x // 3) % 4 * 60).astype(np.uint8), (50, 60, 3)).copy()
        K, D, C = 11, 12, 3
    kn = np.ones(img.shape[:2], np.uint8)
    kn[img.shape[0] // 3: img.shape[0] // 3 + 6, 10:18] = 0
    mi = zb.MultiIndex(img, kn, zb.index_config(patch_size=K, dims=D))
    pm, pc = pca_of(mi)
    om = oracle.MultiIndex(img, kn, K, 0.6, D, pca_mean=pm, pca_comp=pc)
    for l in range(8):
        c, k = mi.index_arrays(l)
        ref = om.index(l)
        lay = mi.layout(l)
        assert np.array_equal(lay["lo"], ref.lo) and np.array_equal(lay["hi"], ref.hi), (case, l)
        assert np.array_equal(c, ref.coords) and np.array_equal(k, ref.keys), (case, l)


def test_pca_householder_path_still_green():
    """The Lanczos fast path delivers the PCA models on every config here, so re-run the PCA and
    build parity tests with it disabled (ZI_PCA_LZ=0): the Householder path (k_pca_tri +
    k_pca_vec), which the fast path falls back to, stays within the same tolerances."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ZI_PCA_LZ="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k",
                        "pca_matches or pca_rgb or build_bitexact or cfg1_end_to_end",
                        os.path.join(root, "tests", "test_gpu_parity.py")],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_sharded_build_with_empty_shards(zb):
    """More ranks than dictionary patches: the empty slices take part in every collective with
    identity ranges and sentinel samples; the non-empty shards still equal the single-GPU build."""
    rng = np.random.default_rng(41)
    img = rng.integers(0, 256, (11, 13), dtype=np.uint8)  # K = 9: 3 x 5 = 15 windows
    kn = np.ones_like(img)
    kn[0, 4] = 0  # removes the windows covering (0, 4)
    cfg = zb.index_config(patch_size=9, dims=4, knn=4)
    mi = zb.MultiIndex(img, kn, cfg)
    world = mi.n + 3
    sharding, shards, _ = _sharded(zb, img, kn, cfg, world, samples=4)
    ranges = sharding.shard_ranges(mi.n, world)
    assert any(e == b for b, e in ranges)
    for l in range(8):
        c, k = mi.index_arrays(l)
        cs = np.concatenate([sh.multi_index.index_arrays(l)[0] for sh in shards])
        ks = np.concatenate([sh.multi_index.index_arrays(l)[1] for sh in shards])
        assert np.array_equal(cs, c) and np.array_equal(ks, k), l


def test_moments_patch_matrix_path_still_green():
    """The fused tensor-core moments cover every configuration here; re-run the moment and build
    parity tests on the patch-matrix + TMA Gram path (ZI_MOMENTS_TMA=1), the fallback for patch
    shapes outside the fused kernel's envelope."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ZI_MOMENTS_TMA="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k",
                        "moments_exact or build_bitexact or cfg1_end_to_end",
                        os.path.join(root, "tests", "test_gpu_parity.py")],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# ------------------------------------------------------------------ build_index / make_query / brute force (C ABI)
@pytest.mark.parametrize("case", range(4))
def test_build_index_one_layout_vs_oracle(zb, golden, case):
    """zi_index_build (build_index, builder.hpp:77-81) over a caller dictionary and layout: the
    device model injected into the oracle restatement gives the same lo / hi, coords and keys;
    on the multi-index's dictionary and layouts the model and bytes equal the multi-index's."""
    tag, img, kn = _images(golden)[case]
    C = 1 if img.ndim == 2 else img.shape[2]
    cfg = zb.index_config(patch_size=9, dims=8)
    mi = zb.MultiIndex(img, kn, cfg)
    d = mi.dictionary
    for l in (0, 4, 7):
        lay = mi.layout(l)
        pi = zb.PatchIndex(img, d, lay["pixels"], cfg)
        mod = pi.model()
        assert np.array_equal(mod["mean"], lay["mean"]), (tag, l)
        np.testing.assert_allclose(mod["components"], lay["components"], atol=1e-9)
        lo, hi, coords, _ = oracle.project_build(img, d, lay["pixels"], mod["mean"], mod["components"])
        assert np.array_equal(lo, mod["lo"]) and np.array_equal(hi, mod["hi"]), (tag, l)
        rc, rk = oracle.from_descriptors(coords, d)
        c, k = pi.index().export()
        assert np.array_equal(c, rc) and np.array_equal(k, rk), (tag, l)
        if np.array_equal(mod["components"], lay["components"]):
            assert np.array_equal(c, mi.index_arrays(l)[0]) and np.array_equal(k, mi.index_arrays(l)[1])
        for tv, tk in _query_cases(img, kn, 11):
            q = pi.make_query(tv, tk)
            assert np.array_equal(q, oracle.make_query(tv, tk, 9, C, lay["pixels"], mod["mean"], mod["components"],
                                                       lo, hi)), (tag, l)
            # the multi-index layout's make_query, same arithmetic
            mq = mi.make_query(l, tv, tk)
            assert np.array_equal(mq, oracle.make_query(tv, tk, 9, C, lay["pixels"], lay["mean"], lay["components"],
                                                        lay["lo"], lay["hi"]))


def test_build_index_custom_layout_and_subset_dictionary(zb, golden):
    """A layout that is not one of the eight (the first 30 row-major offsets) over every third
    dictionary key; D clamps to min(dims, m*C, n)."""
    img, kn = workloads.small_image(64, 80, 3, seed=5, hole_frac=0.08)
    cfg = zb.index_config(patch_size=7, dims=12)
    d = oracle.collect_dictionary(kn, 7)[::3].copy()
    rc = np.array([(i // 7, i % 7) for i in range(30)], dtype=np.int32)
    pi = zb.PatchIndex(img, d, rc, cfg)
    mod = pi.model()
    assert pi.dims == 12 and pi.mc == 90
    lo, hi, coords, _ = oracle.project_build(img, d, rc, mod["mean"], mod["components"])
    assert np.array_equal(lo, mod["lo"]) and np.array_equal(hi, mod["hi"])
    c, k = pi.index().export()
    rcs, rks = oracle.from_descriptors(coords, d)
    assert np.array_equal(c, rcs) and np.array_equal(k, rks)
    tiny = zb.PatchIndex(img, d[:3], rc, cfg)
    assert tiny.dims == 3
    with pytest.raises(zb.EmptyDictionaryError):
        zb.PatchIndex(img, d[:0], rc, cfg)
    with pytest.raises(ValueError):
        zb.PatchIndex(img, np.array([(63 << 16) | 79], np.uint32), rc, cfg)  # window outside the image


@pytest.mark.parametrize("norm", ["l2", "l1"])
def test_brute_force_scan_caller_dictionary(zb, golden, norm):
    """zi_brute_force_scan (brute_force_best(image, target, dictionary, norm)) over a subset of the
    dictionary equals the oracle's scan of the same subset."""
    tag, img, kn = _images(golden)[1]
    d = oracle.collect_dictionary(kn, 9)
    sub = d[(np.arange(d.size) % 5) != 2].copy()
    nrm = L2 if norm == "l2" else L1
    for tv, tk in _query_cases(img, kn, 6):
        key, cost, _ = zb.brute_force_scan(img, sub, tv, tk, 9, norm)
        assert (cost << 32 | key) == oracle.brute_force_best(img, tv, tk, 9, sub, nrm)


def _device_shard_worker(rank, world, port, q):
    """One rank of a 2-process sharded build on the device (zi_shard_* stages), exchanging over
    gloo with host staging -- both ranks share the one GPU, no kernel waits on the other rank."""
    import os

    import torch
    import torch.distributed as dist

    import paper_1712_06326_b200 as zb
    from paper_1712_06326_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        img, known = workloads.small_image(96, 120, 3, seed=23, hole_frac=0.07)
        cfg = zb.index_config(patch_size=7, dims=8, knn=24)
        sh = sharding.DeviceShard(img, known, cfg, rank, world)
        info = sharding.build_sharded([sh], sharding.TorchComm(), samples=64)
        first = {l: sh.multi_index.index_arrays(l) for l in range(8)}
        sh.rebuild()  # the buffers are kept; the second build must give the same bytes
        sharding.build_sharded([sh], sharding.TorchComm(), samples=64)
        same = all(np.array_equal(first[l][0], sh.multi_index.index_arrays(l)[0]) and
                   np.array_equal(first[l][1], sh.multi_index.index_arrays(l)[1]) for l in range(8))
        mi = zb.MultiIndex(img, known, cfg)
        b, e = sharding.shard_ranges(mi.n, world)[rank]
        ok = same and (sh.row_begin, sh.row_end) == (b, e)
        for l in range(8):
            c, k = mi.index_arrays(l)
            cs, ks = first[l]
            ok = ok and np.array_equal(cs, c[b:e]) and np.array_equal(ks, k[b:e])
        # the sharded query over gloo equals the single-GPU query
        for (x, y) in fillfront(known)[:6]:
            tv, tk = oracle.extract_patch_clamped(img, known, int(x), int(y), 7)
            got = sharding.sharded_query([sh], sharding.TorchComm(), tv, tk, 24, 0)[0]
            want = mi.query_best_patch(tv, tk)
            ok = ok and (got[0], got[1], got[3], got[4]) == (want[0], want[1], want[3], want[4])
        q.put((rank, bool(ok), info["records_exchanged"]))
    except Exception as ex:  # noqa: BLE001
        q.put((rank, repr(ex), 0))
    finally:
        dist.destroy_process_group()


def test_sharded_build_device_gloo_world2():
    """Two processes run the device zi_shard_* stages end to end (NCCL stands in for gloo with
    host staging: the pool has one GPU) and each holds exactly its slice of the single-GPU build."""
    import multiprocessing as mp

    from tests.test_cpu import _free_port
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_device_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(g[1] is True for g in got), got
    assert got[0][2] > 0


def test_sharded_world1_local_finish_and_rebuild(zb):
    """World 1 skips the exchange (finish_local) and a rebuild keeps the buffers: both equal the
    single-GPU build byte for byte."""
    from paper_1712_06326_b200 import sharding
    img, known = workloads.small_image(80, 100, 1, seed=29, hole_frac=0.08)
    cfg = zb.index_config(patch_size=9, dims=8, knn=16)
    mi = zb.MultiIndex(img, known, cfg)
    sh = sharding.DeviceShard(img, known, cfg, 0, 1)
    info = sharding.build_sharded([sh], sharding.LoopbackComm(1))
    assert info["records_exchanged"] == 0
    for rep in range(2):
        for l in range(8):
            a, b = sh.multi_index.index_arrays(l), mi.index_arrays(l)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), (rep, l)
        sh.rebuild()
        sharding.build_sharded([sh], sharding.LoopbackComm(1))
