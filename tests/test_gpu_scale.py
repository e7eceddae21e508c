"""GPU parity at the configs' full sizes (SURVEY.md §8(c) parity matrix).

Every artifact is compared byte for byte -- no sampling:

* cfg2 (n = 950,771, K = 11, RGB, D = 12) and cfg4 (n = 14.9 M, K = 9, D = 8): all 8 layouts'
  quantised coords, keys and quantiser lo / hi against the oracle restatement of
  ``build_index`` (proj/src/builder.cpp:129-195) fed the device PCA model;
* the sort permutation of one layout at cfg2 and cfg4 against the reference's OWN compiled
  ``zcurve_index::from_descriptors`` (proj/src/zcurve.cpp:108-138, oracle/_ref/libzref.so);
* the whole cfg2 fill loop and the first 2,000 cfg4 iterations against the restated
  ``run_loop`` (proj/src/engine.cpp:371-438): targets, layouts, source keys, costs, and the
  final cfg2 image;
* cfg5 (BASELINE configs[4]) at n = 2^20, D in {4, 8, 16}: mean / covariance, quantiser ranges
  and coords of the vector build, its sort against the compiled ``from_descriptors``, and 256
  k-NN lists against the compiled ``knn_search`` (proj/src/zcurve.cpp:429-452).

The oracle runs on the GPU box's host cores (layouts and scans split over threads; the results
do not depend on the split).
"""
import os
import threading

import numpy as np
import pytest

import oracle
import workloads
from tests.helpers import pca_of

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

L2 = 0


def _threads(n=8):
    return max(1, min(n, os.cpu_count() or 1))


def _run_parallel(fns):
    """Run callables on Python threads (the oracle calls release the GIL); re-raise failures."""
    out, errs = [None] * len(fns), []

    def wrap(i, f):
        try:
            out[i] = f()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=wrap, args=(i, f)) for i, f in enumerate(fns)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def _unsorted(coords, keys, dictionary):
    """A layout's descriptors back in dictionary (row-major key) order: the input the reference's
    from_descriptors receives from build_index (proj/src/builder.cpp:177-187)."""
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(keys[order], dictionary)
    return coords[order]


def _compare_runs(recs, rrecs, n=None):
    n = len(rrecs) if n is None else n
    assert len(recs) >= n and len(rrecs) >= n
    r, o = recs[:n], rrecs[:n]
    assert np.array_equal(r["target_x"], o["tx"]) and np.array_equal(r["target_y"], o["ty"])
    assert np.array_equal(r["layout_id"], o["layout_id"])
    assert np.array_equal(r["source_key"], (o["sy"].astype(np.uint32) << 16) | o["sx"].astype(np.uint32))
    assert np.array_equal(r["cost"], o["cost"])
    assert np.array_equal(r["candidates"], o["candidates"])


def _check_layouts(mi, om, layouts):
    for l in layouts:
        c, k = mi.index_arrays(l)
        ref = om.index(l)
        lay = mi.layout(l)
        assert np.array_equal(lay["lo"].view(np.uint64), ref.lo.view(np.uint64)), l
        assert np.array_equal(lay["hi"].view(np.uint64), ref.hi.view(np.uint64)), l
        assert np.array_equal(c, ref.coords), l
        assert np.array_equal(k, ref.keys), l


# ------------------------------------------------------------------ cfg2
@pytest.fixture(scope="module")
def cfg2_pair(zb):
    img, kn, p = workloads.cfg2()
    mi = zb.MultiIndex(img, kn, zb.index_config(**p))
    pm, pc = pca_of(mi)
    om = oracle.MultiIndex(img, kn, p["patch_size"], 0.6, p["dims"], pca_mean=pm, pca_comp=pc,
                           threads=_threads())
    return img, kn, p, mi, om


def test_cfg2_all_layouts_bitexact(cfg2_pair):
    img, kn, p, mi, om = cfg2_pair
    assert mi.n == om.n == 950771
    assert np.array_equal(mi.dictionary, om.dictionary())
    _check_layouts(mi, om, range(8))


def test_cfg2_sort_equals_compiled_reference(cfg2_pair):
    img, kn, p, mi, om = cfg2_pair
    for l in (0, 5):
        c, k = mi.index_arrays(l)
        rc, rk = oracle.ref_from_descriptors(_unsorted(c, k, mi.dictionary), mi.dictionary)
        assert np.array_equal(c, rc) and np.array_equal(k, rk), l


def test_cfg2_fill_loop_bitexact(cfg2_pair):
    """The whole cfg2 run (~1.9k iterations): every record and the final image."""
    img, kn, p, mi, om = cfg2_pair
    out, recs, stats = mi.inpaint()
    rout, rrecs = oracle.inpaint(img, kn, p["patch_size"], 0.6, p["dims"], knn=p["knn"], mi=om)
    assert len(recs) == len(rrecs) > 1000
    _compare_runs(recs, rrecs)
    assert np.array_equal(out, rout)
    known = kn != 0
    assert np.array_equal(out[known], img[known])


# ------------------------------------------------------------------ cfg4
@pytest.fixture(scope="module")
def cfg4_pair(zb):
    img, kn, p = workloads.cfg4()
    mi = zb.MultiIndex(img, kn, zb.index_config(**p))
    pm, pc = pca_of(mi)
    om = oracle.MultiIndex(img, kn, p["patch_size"], 0.6, p["dims"], pca_mean=pm, pca_comp=pc,
                           threads=_threads())
    return img, kn, p, mi, om


def test_cfg4_all_layouts_bitexact(cfg4_pair):
    img, kn, p, mi, om = cfg4_pair
    assert mi.n == om.n == 14915904
    assert np.array_equal(mi.dictionary, om.dictionary())
    _check_layouts(mi, om, range(8))


def test_cfg4_rebuild_fused_sort_bitexact(cfg4_pair):
    """The first cfg4 build finds the top Morton bytes too clustered for the MSD split and falls
    back to LSD; later builds go straight to LSD passes whose last pass writes the indices (the
    bench's steady state).  That rebuild is byte-equal to the oracle too."""
    img, kn, p, mi, om = cfg4_pair
    mi.ctx.set_profiling(True)
    mi.rebuild()
    prof = mi.ctx.profile()
    mi.ctx.set_profiling(False)
    assert prof.get("index_bbox", (0.0, 0))[1] == 1 and prof.get("finalize_index", (0.0, 0))[1] == 0
    _check_layouts(mi, om, range(8))


def test_cfg4_sort_equals_compiled_reference(cfg4_pair):
    img, kn, p, mi, om = cfg4_pair
    d = mi.dictionary
    jobs = []
    for l in (3,):
        c, k = mi.index_arrays(l)
        u = _unsorted(c, k, d)
        jobs.append(lambda u=u: oracle.ref_from_descriptors(u, d))
    got = _run_parallel(jobs)
    for l, (rc, rk) in zip((3,), got):
        c, k = mi.index_arrays(l)
        assert np.array_equal(c, rc) and np.array_equal(k, rk), l


def test_cfg4_fill_loop_prefix_bitexact(cfg4_pair):
    """The first 2,000 iterations of the cfg4 run (of ~48k) equal the oracle's."""
    img, kn, p, mi, om = cfg4_pair
    out, recs, stats = mi.inpaint()
    rout, rrecs = oracle.inpaint(img, kn, p["patch_size"], 0.6, p["dims"], knn=p["knn"], mi=om, max_iter=2000)
    assert len(rrecs) == 2000
    _compare_runs(recs, rrecs, 2000)
    known = kn != 0
    assert np.array_equal(out[known], img[known])
    assert stats.iterations == len(recs)


# ------------------------------------------------------------------ cfg5 at n = 2^20
@pytest.fixture(scope="module")
def cfg5_data():
    n = 1 << 20
    X = workloads.cfg5_points(n, dims_in=125, seed=5)
    mean, cov = oracle.vec_mean_cov(X)
    rng = np.random.default_rng(6)
    Q = workloads.cfg5_points(256, dims_in=125, seed=66)
    known = (rng.random(Q.shape) >= 0.4).astype(np.uint8)
    return X, mean, cov, Q, known


@pytest.mark.parametrize("D", [4, 8, 16])
def test_cfg5_vector_build_and_knn_vs_compiled_reference(zb, cfg5_data, D):
    X, mean, cov, Q, known = cfg5_data
    n = X.shape[0]
    vi = zb.VectorIndex(X, D)
    mod = vi.model()
    assert np.array_equal(mod["mean"], mean)
    comp, eig = oracle.pca_from_cov(cov, D)
    np.testing.assert_allclose(mod["eigenvalues"], eig, rtol=1e-9, atol=1e-9 * eig[0])
    Cm = mod["components"]
    lo, hi, coords = oracle.vec_project(X, mod["mean"], Cm)
    assert np.array_equal(lo.view(np.uint64), mod["lo"].view(np.uint64))
    assert np.array_equal(hi.view(np.uint64), mod["hi"].view(np.uint64))
    rows = np.arange(n, dtype=np.uint32)
    ref = oracle.RefIndex(coords, rows)  # the reference's from_descriptors
    rc, rk = ref.export()
    c, k = vi.index().export()
    assert np.array_equal(c, rc) and np.array_equal(k, rk)
    qd = vi.make_queries(Q, known)
    for i in range(0, Q.shape[0], 17):
        assert np.array_equal(qd[i], oracle.vec_make_query(Q[i], known[i], mod["mean"], Cm, lo, hi))
    out, cnt = vi.knn(Q, known, k=80)
    want, wcnt = ref.knn_batch(qd, 80, threads=_threads(16))
    assert np.array_equal(cnt, wcnt)
    assert np.array_equal(out, want)
