"""CPU suite (no GPU): the oracle pinned against the reference's own vectors and known answers,
the host logic behind the C ABI, the ABI's symbol table, and the multi-rank (gloo) logic."""
import ctypes as C
import os
import re
import socket

import numpy as np
import pytest

import oracle
import workloads
from tests.helpers import fillfront, morton_words

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L2, L1 = 0, 1


# ------------------------------------------------------------------ Morton order
def test_msb_table_exhaustive():
    """test_morton.cpp:11-20"""
    def msb(v):
        return v.bit_length() - 1
    for a in range(256):
        for b in range(256):
            assert oracle.lib().zo_less_msb(a, b) == (msb(a) < msb(b))


def test_morton_known_answer():
    """z(3,0)=10 < z(2,3)=13 (test_morton.cpp:27-35)"""
    a = np.array([3, 0], np.uint8)
    b = np.array([2, 3], np.uint8)
    assert oracle.morton_less(a, b) and not oracle.morton_less(b, a)
    w = morton_words(np.array([[3, 0], [2, 3]], np.uint8))[0]
    # 8-bit interleave: the 4-bit z-values of the test sit in the low bits
    assert int(w[0]) & 0xF == 10 and int(w[1]) & 0xF == 13


@pytest.mark.parametrize("D", [2, 4, 8, 16])
def test_morton_pairs_match_reference(golden, D):
    a, b, less = (golden[f"morton_D{D}__{x}"] for x in ("a", "b", "less"))
    got = np.array([oracle.morton_less(a[i], b[i]) for i in range(len(less))])
    assert np.array_equal(got, less.astype(bool))
    wa, wb = morton_words(a), morton_words(b)
    lt = np.zeros(len(less), bool)
    eq = np.ones(len(less), bool)
    for x, y in zip(wa, wb):
        lt |= eq & (x < y)
        eq &= x == y
    assert np.array_equal(lt, less.astype(bool))  # explicit interleave oracle (oracles.hpp:33-39)


# ------------------------------------------------------------------ z-curve sort + knn
@pytest.mark.parametrize("kind", ["uniform", "clustered"])
@pytest.mark.parametrize("D", [4, 8, 10, 16])
def test_oracle_from_descriptors_golden(golden, kind, D):
    tag = f"{kind}_D{D}"
    c, k = oracle.from_descriptors(golden[tag + "__coords"], np.arange(golden[tag + "__coords"].shape[0],
                                                                       dtype=np.uint32))
    assert np.array_equal(c, golden[tag + "__sorted_coords"])
    assert np.array_equal(k, golden[tag + "__sorted_keys"])


@pytest.mark.parametrize("kind", ["uniform", "clustered"])
@pytest.mark.parametrize("D", [4, 8, 10, 16])
def test_oracle_knn_golden(golden, kind, D):
    tag = f"{kind}_D{D}"
    sc, sk = golden[tag + "__sorted_coords"], golden[tag + "__sorted_keys"]
    for nname, norm in (("l2", L2), ("l1", L1)):
        for k in (1, 10, 80):
            ref = golden[f"{tag}__knn_{nname}_k{k}"]
            for qi, q in enumerate(golden[tag + "__queries"]):
                assert np.array_equal(oracle.knn_linear(sc, sk, q, k, norm), ref[qi])


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_compiled_reference_matches_golden(golden):
    R = oracle.ref()
    tag = "clustered_D8"
    coords = golden[tag + "__coords"]
    keys = np.arange(coords.shape[0], dtype=np.uint32)
    h = R.zr_index_create(coords.ctypes.data_as(C.POINTER(C.c_uint8)), keys.ctypes.data_as(C.POINTER(C.c_uint32)),
                          coords.shape[0], 8)
    c = np.zeros_like(coords)
    k = np.zeros_like(keys)
    R.zr_index_export(h, c.ctypes.data_as(C.POINTER(C.c_uint8)), k.ctypes.data_as(C.POINTER(C.c_uint32)))
    R.zr_index_free(h)
    assert np.array_equal(c, golden[tag + "__sorted_coords"]) and np.array_equal(k, golden[tag + "__sorted_keys"])


def test_oracle_sort_unsorted_keys_and_ties():
    rng = np.random.default_rng(1)
    coords = (rng.integers(0, 4, (3000, 3)) * 60).astype(np.uint8)
    keys = rng.permutation(3000).astype(np.uint32)
    c, k = oracle.from_descriptors(coords, keys)
    words = morton_words(c)
    order = np.lexsort([k] + words[::-1])
    assert np.array_equal(order, np.arange(3000))


# ------------------------------------------------------------------ layouts
def test_layouts_match_reference(golden):
    for K in (3, 5, 7, 9, 11, 13):
        for c in (0.25, 0.6, 1.0):
            ref = golden[f"layouts_K{K}_c{int(c * 100 + 0.5):03d}"]
            assert np.array_equal(oracle.subset_layouts(K, c), ref)


def test_layout_union_covers_patch():
    """proj/tests/python/test_smoke.py:25-34"""
    lay = oracle.subset_layouts(9, 0.6)
    assert lay.shape == (8, 49, 2)
    assert len({(int(r), int(c)) for l in lay for r, c in l}) == 81


# ------------------------------------------------------------------ quantiser (test_pca.cpp:101-141)
def test_quantizer_known_answers():
    assert oracle.quantize(-2.0, 2.0, -2.0) == 0
    assert oracle.quantize(-2.0, 2.0, 2.0) == 255
    assert oracle.quantize(-2.0, 2.0, 1.0) == 191
    assert oracle.quantize(-2.0, 2.0, -5.0) == 0
    assert oracle.quantize(-2.0, 2.0, 7.0) == 255
    assert oracle.quantize(1.0, 1.0, 1.0) == 0 and oracle.quantize(1.0, 1.0, 99.0) == 0
    prev = 0
    for y in np.arange(-5.0, 13.0, 0.01):
        b = oracle.quantize(-3.7, 11.2, y)
        assert b >= prev
        prev = b
    assert oracle.quantize(-4.0, 4.0, 0.0) == 128  # the mean maps to round(255/2)


# ------------------------------------------------------------------ PCA (test_pca.cpp:11-99 protocols)
def test_pca_axis_aligned():
    rng = np.random.default_rng(67)
    x = rng.normal(size=(4000, 3)) * np.array([9.0, 3.0, 0.5])
    comp, eig = oracle.pca_from_cov(np.cov(x.T), 3)
    assert eig[0] >= eig[1] >= eig[2]
    for j in range(3):
        assert abs(comp[j, j]) > 0.99 and comp[j, j] > 0
    np.testing.assert_allclose(comp @ comp.T, np.eye(3), atol=1e-10)


def test_pca_diagonal_known_answer():
    x = np.array([[0, 0], [2, 2], [4, 4]], float)
    s = x.sum(0).astype(np.int64)
    S = (x.T @ x).astype(np.int64)
    mean, cov = oracle.layout_covariance(s, S, 3, np.array([0, 1], np.int32))
    assert np.array_equal(mean, [2.0, 2.0])
    comp, eig = oracle.pca_from_cov(cov, 1)
    np.testing.assert_allclose(comp[0], [2 ** -0.5, 2 ** -0.5], rtol=1e-12)
    np.testing.assert_allclose(eig[0], 8.0, rtol=1e-12)


def test_pca_identical_samples_zero_eigenvalues():
    s = np.array([40, 10, 25], np.int64) * 10
    S = np.outer([40, 10, 25], [40, 10, 25]).astype(np.int64) * 10
    mean, cov = oracle.layout_covariance(s, S, 10, np.arange(3, dtype=np.int32))
    assert np.array_equal(mean, [40.0, 10.0, 25.0])
    _, eig = oracle.pca_from_cov(cov, 2)
    assert np.all(eig == 0.0)


def test_pca_reconstruction_monotone():
    rng = np.random.default_rng(71)
    lat = rng.normal(size=(500, 2)) * [5, 2]
    j = np.arange(8)
    x = lat[:, :1] * np.sin(0.3 * j) + lat[:, 1:] * np.cos(0.7 * j) + 0.3 * rng.normal(size=(500, 8))
    cov = np.cov(x.T)
    prev = np.inf
    for d in range(1, 9):
        comp, _ = oracle.pca_from_cov(cov, d)
        xc = x - x.mean(0)
        mse = ((xc - xc @ comp.T @ comp) ** 2).sum() / 500
        assert mse <= prev + 1e-9
        prev = mse


def test_moments_exact_small():
    img, kn = workloads.small_image(30, 34, 3, seed=5)
    keys = oracle.collect_dictionary(kn, 5)
    s, S = oracle.patch_moments(img, 5, keys)
    X = np.stack([img[(k >> 16):(k >> 16) + 5, (k & 0xFFFF):(k & 0xFFFF) + 5].reshape(-1) for k in keys]).astype(np.int64)
    assert np.array_equal(s, X.sum(0)) and np.array_equal(S, X.T @ X)


# ------------------------------------------------------------------ dictionary (test_builder.cpp:10-39)
def test_dictionary_counts(golden):
    known = np.ones((20, 20), np.uint8)
    assert oracle.collect_dictionary(known, 9).size == 144
    assert oracle.collect_dictionary(np.zeros((20, 20), np.uint8), 9).size == 0
    holed = known.copy()
    holed[10, 10] = 0
    keys = oracle.collect_dictionary(holed, 9)
    assert keys.size == 144 - 81
    expect = [(y << 16) | x for y in range(12) for x in range(12) if holed[y:y + 9, x:x + 9].all()]
    assert np.array_equal(keys, expect)


def test_workload_sizes():
    img, kn, _ = workloads.cfg1()
    assert img.shape == (256, 256) and oracle.collect_dictionary(kn, 9).size == 58368


# ------------------------------------------------------------------ costs and selection (test_engine.cpp)
def test_masked_cost_known_answers():
    tv = np.zeros(9, np.uint8)
    tk = np.zeros(9, np.uint8)
    img = np.zeros((3, 3), np.uint8)
    assert oracle.masked_cost_at(img, tv, tk, 3, 0) == 0
    tk[4], tv[4], img[1, 1] = 1, 10, 5
    assert oracle.masked_cost_at(img, tv, tk, 3, 0, L2) == 25
    assert oracle.masked_cost_at(img, tv, tk, 3, 0, L1) == 5
    img[1, 1], img[0, 0] = 10, 200
    assert oracle.masked_cost_at(img, tv, tk, 3, 0) == 0


def test_select_index_known_answers():
    lay = oracle.subset_layouts(9, 0.6)
    full = np.ones(81, np.uint8)
    assert oracle.lib().zo_select_index(full.ctypes.data_as(C.POINTER(C.c_uint8)), 9,
                                        lay.ctypes.data_as(C.POINTER(C.c_int)), 49) == 0
    left = np.zeros((9, 9), np.uint8)
    left[:, :4] = 1
    left = left.reshape(-1).copy()
    assert oracle.lib().zo_select_index(left.ctypes.data_as(C.POINTER(C.c_uint8)), 9,
                                        lay.ctypes.data_as(C.POINTER(C.c_int)), 49) == 3
    tight = oracle.subset_layouts(9, 0.25)
    tl = np.zeros((9, 9), np.uint8)
    tl[:4, :4] = 1
    tl = tl.reshape(-1).copy()
    assert oracle.lib().zo_select_index(tl.ctypes.data_as(C.POINTER(C.c_uint8)), 9,
                                        tight.ctypes.data_as(C.POINTER(C.c_int)), tight.shape[1]) == 4


def test_priority_known_answers():
    """test_engine.cpp:69-125"""
    img = np.full((21, 21), 77, np.uint8)
    known = np.ones((21, 21), np.uint8)
    known[:, 11:] = 0
    conf = known.astype(float)
    p = oracle.compute_priority(img, known, conf, 10, 10, 9)
    assert p == pytest.approx(1e-3 * 45.0 / 81.0)
    k2 = np.ones((21, 21), np.uint8)
    k2[10, 10] = 0
    c2 = np.ones((21, 21))
    c2[10, 10] = 0
    assert oracle.confidence_term(k2, c2, 10, 10, 9) == pytest.approx(80.0 / 81.0)
    w = h = 24
    step = np.where(np.arange(h)[:, None] < 12, 40, 200).repeat(w, 1).astype(np.uint8)
    km = np.ones((h, w), np.uint8)
    km[:, 12:] = 0
    cf = km.astype(float)
    conf_t = oracle.confidence_term(km, cf, 11, 11, 9)
    assert oracle.compute_priority(step, km, cf, 11, 11, 9) == pytest.approx(conf_t * (80.0 / 255.0 + 1e-3))
    par = np.where(np.arange(w)[None, :] < 6, 40, 200).repeat(h, 0).astype(np.uint8)
    assert oracle.compute_priority(par, km, cf, 11, 11, 9) == pytest.approx(conf_t * 1e-3)


def test_extract_and_fillfront_match_reference(golden):
    for tag in ("eval_64x64_g_s90_m91", "eval_48x40_c_s101_m102"):
        img = golden[tag + "__image"]
        img = img[:, :, 0] if img.shape[2] == 1 else img
        kn = golden[tag + "__known"]
        assert fillfront(kn) == [tuple(p) for p in golden[tag + "__front"].tolist()]
        if oracle.ref_available():
            R = oracle.ref()
            h, w = kn.shape
            ch = 1 if img.ndim == 2 else 3
            for (x, y) in fillfront(kn)[::11]:
                tv, tk = oracle.extract_patch_clamped(img, kn, x, y, 9)
                rv = np.zeros_like(tv)
                rk = np.zeros_like(tk)
                R.zr_extract_patch_clamped(np.ascontiguousarray(img).ctypes.data_as(C.POINTER(C.c_uint8)),
                                           kn.ctypes.data_as(C.POINTER(C.c_uint8)), w, h, ch, x, y, 9,
                                           rv.ctypes.data_as(C.POINTER(C.c_uint8)),
                                           rk.ctypes.data_as(C.POINTER(C.c_uint8)))
                assert np.array_equal(tv, rv) and np.array_equal(tk, rk)


def test_brute_force_exact_match(golden):
    img = golden["eval_30x30_g_s91__image"][:, :, 0]
    kn = np.ones((30, 30), np.uint8)
    kn[20:29, 20:29] = 0
    d = oracle.collect_dictionary(kn, 9)
    tv, tk = oracle.extract_patch_clamped(img, np.ones((30, 30), np.uint8), 6, 6, 9)
    assert oracle.brute_force_best(img, tv, tk, 9, d) == (2 << 16 | 2)


# ------------------------------------------------------------------ the oracle fill loop
def _naive_loop(img, kn, mi, K, k):
    """test_engine.cpp:383-427: recompute the front and priorities from scratch each step."""
    img = img.copy()
    kn = kn.copy()
    conf = kn.astype(float)
    targets, sources = [], []
    while (kn == 0).any():
        front = fillfront(kn)
        pr = [oracle.compute_priority(img, kn, conf, x, y, K) for x, y in front]
        best = 0
        for i in range(1, len(front)):
            if pr[i] > pr[best] or (pr[i] == pr[best] and (front[i][1], front[i][0]) < (front[best][1], front[best][0])):
                best = i
        x, y = front[best]
        tv, tk = oracle.extract_patch_clamped(img, kn, x, y, K)
        packed, *_ = mi.query_best_patch(img, tv, tk, k)
        src = packed & 0xFFFFFFFF
        sx, sy = src & 0xFFFF, src >> 16
        cc = oracle.confidence_term(kn, conf, x, y, K)
        r = (K - 1) // 2
        for dy in range(K):
            for dx in range(K):
                yy, xx = y - r + dy, x - r + dx
                if 0 <= yy < kn.shape[0] and 0 <= xx < kn.shape[1] and not kn[yy, xx]:
                    img[yy, xx] = img[sy + dy, sx + dx]
                    kn[yy, xx] = 1
                    conf[yy, xx] = cc
        targets.append((x, y))
        sources.append(int(src))
    return img, targets, sources


def test_oracle_engine_equals_naive_loop(golden):
    img = golden["eval_32x28_g_s103_m104__image"][:, :, 0]
    kn = golden["eval_32x28_g_s103_m104__known"]
    mi = oracle.MultiIndex(img, kn, 9, 0.6, 6)
    out, recs = oracle.inpaint(img, kn, 9, 0.6, 6, knn=10, mi=mi)
    nimg, targets, sources = _naive_loop(img, kn, mi, 9, 10)
    assert [(int(r["tx"]), int(r["ty"])) for r in recs] == targets
    assert [int(r["sy"]) << 16 | int(r["sx"]) for r in recs] == sources
    assert np.array_equal(out, nimg)


def test_oracle_inpaint_conservation_and_oracle_mode(golden):
    img = golden["eval_36x30_g_s105_m106__image"][:, :, 0]
    kn = golden["eval_36x30_g_s105_m106__known"]
    out, recs = oracle.inpaint(img, kn, 9, 0.6, 6, knn=4, oracle=True)
    assert len(recs) > 0 and (recs["z_error"] >= recs["bf_error"]).all()
    assert np.array_equal(out[kn != 0], img[kn != 0])


# ------------------------------------------------------------------ the C ABI (no compute calls)
def _header_functions():
    text = open(os.path.join(ROOT, "include", "zinpaint_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(zi_[a-z0-9_]+)\s*\(", text)))


def test_abi_exports_every_declared_symbol():
    import paper_1712_06326_b200._lib as L
    lib = L.lib()
    names = _header_functions()
    assert len(names) >= 35
    for name in names:
        assert hasattr(lib, name), name
        assert name in L.SIGNATURES, f"{name} missing from the ctypes signature table"


def test_abi_host_utilities_match_oracle(golden):
    import paper_1712_06326_b200 as zb
    a, b, less = golden["morton_D8__a"], golden["morton_D8__b"], golden["morton_D8__less"]
    for i in range(0, len(less), 7):
        assert zb.morton_less(a[i], b[i]) == bool(less[i])
    for x in range(0, 256, 5):
        for y in range(0, 256, 3):
            assert zb.less_most_significant_bit(x, y) == bool(oracle.lib().zo_less_msb(x, y))
    for K in (3, 9, 11):
        for c in (0.25, 0.6):
            got = np.array([l["pixels"] for l in zb.subset_layouts(K, c)])
            assert np.array_equal(got, golden[f"layouts_K{K}_c{int(c * 100 + 0.5):03d}"])


def test_abi_config_validation():
    """index_config::validate (test_builder.cpp:115-133)"""
    import paper_1712_06326_b200 as zb
    L = zb._lib.lib()
    ok = zb.index_config()
    assert L.zi_index_config_validate(C.byref(ok), 3) == 0
    for kw in (dict(patch_size=8), dict(coverage=0.0), dict(dims=0), dict(dims=500), dict(nu=4), dict(knn=0)):
        bad = zb.index_config(**kw)
        assert L.zi_index_config_validate(C.byref(bad), 3) == zb._lib.ZI_E_INVALID, kw


# ------------------------------------------------------------------ multi-rank logic (gloo, world 2)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1712_06326_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        n, D, k = 20000, 8, 80
        coords = rng.integers(0, 256, (n, D)).astype(np.uint8)
        keys = np.arange(n, dtype=np.uint32)
        sc, sk = oracle.from_descriptors(coords, keys)
        b, e = sharding.shard_ranges(n, world)[rank]
        res = []
        for t in range(5):
            qv = rng.integers(0, 256, D).astype(np.uint8)
            local = oracle.knn_linear(sc[b:e], sk[b:e], qv, k)  # stands in for the shard's GPU top-k
            merged = sharding.allgather_topk(local, k)
            res.append(bool(np.array_equal(merged, oracle.knn_linear(sc, sk, qv, k))))
            # brute-force winners min-reduced as packed u64
            val = int(local[0]) if local.size else np.iinfo(np.int64).max
            res.append(sharding.allreduce_min_packed(val) == int(oracle.knn_linear(sc, sk, qv, 1)[0]))
        q.put((rank, all(res)))
    finally:
        dist.destroy_process_group()


def test_sharded_query_merge_gloo_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert out == {0: True, 1: True}


def test_shard_ranges_cover():
    from paper_1712_06326_b200 import sharding
    for n in (0, 1, 7, 1000, 1001):
        for w in (1, 2, 3, 8):
            r = sharding.shard_ranges(n, w)
            assert r[0][0] == 0 and r[-1][1] == n and all(r[i][1] == r[i + 1][0] for i in range(w - 1))
    lists = [np.array([5, 9], np.uint64), np.array([1, 7, 8], np.uint64), np.array([], np.uint64)]
    assert np.array_equal(sharding.merge_topk(lists, 3), [1, 5, 7])


# ------------------------------------------------------------------ sharded build (§8(e)) on CPU
def _shard_case():
    img, known = workloads.small_image(40, 46, 1, seed=3, hole_frac=0.1)
    return img, known, 5, 0.6, 6


def _check_sharded(outs, world):
    """Concatenated shard indices == the oracle's single-host multi_index::build."""
    from paper_1712_06326_b200 import sharding
    img, known, K, cov, D = _shard_case()
    om = oracle.MultiIndex(img, known, K, cov, D)
    ranges = sharding.shard_ranges(om.n, world)
    for l in range(8):
        ref = om.index(l)
        for r in range(world):
            b, e = ranges[r]
            c, k = outs[r][l]
            assert np.array_equal(c, ref.coords[b:e]) and np.array_equal(k, ref.keys[b:e]), (l, r)


def _shard_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1712_06326_b200 import sharding
    from tests.helpers import OracleShard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img, known, K, cov, D = _shard_case()
        sh = OracleShard(img, known, K, cov, D, rank, world)
        info = sharding.build_sharded([sh], sharding.TorchComm(), samples=8)
        q.put((rank, {l: sh.index_arrays(l) for l in range(8)}, info))
    finally:
        dist.destroy_process_group()


def test_sharded_build_gloo_world2():
    """Two processes over gloo run the sample-sort build (moments SUM, lo/hi MIN/MAX, sample
    all-gather, two all-to-alls); rank r holds exactly positions shard_ranges(n, 2)[r]."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    outs = {r: o for r, o, _ in got}
    _check_sharded(outs, 2)
    assert got[0][2]["records_exchanged"] > 0


@pytest.mark.parametrize("world", [1, 3, 5])
def test_sharded_build_loopback_cpu(world):
    from paper_1712_06326_b200 import sharding
    from tests.helpers import OracleShard
    img, known, K, cov, D = _shard_case()
    shards = [OracleShard(img, known, K, cov, D, r, world) for r in range(world)]
    sharding.build_sharded(shards, sharding.LoopbackComm(world), samples=4)
    _check_sharded({r: {l: sh.index_arrays(l) for l in range(8)} for r, sh in enumerate(shards)}, world)


def test_shard_splitters_and_rebalance_plan():
    from paper_1712_06326_b200 import sharding
    rng = np.random.default_rng(9)
    W = 2
    rows = rng.integers(0, 2**32, size=(300, W + 1), dtype=np.uint64).astype(np.uint32)
    rows[:, W] = (rng.integers(0, 8, 300).astype(np.uint32) << 29) | np.arange(300, dtype=np.uint32)
    rows[:5, W] = 0xFFFFFFFF  # "no sample" rows are ignored
    for world in (1, 2, 4, 7):
        sp = sharding.splitters_from_samples([rows], W, world)
        assert sp.shape == (8 * (world - 1), W + 1)
        for l in range(8):
            mine = rows[(rows[:, W] != 0xFFFFFFFF) & ((rows[:, W] >> 29) == l)]
            comp = sorted((int(r[1]) << 64) | (int(r[0]) << 32) | int(r[2]) for r in mine)
            for j in range(1, world):
                r = sp[l * (world - 1) + j - 1]
                assert (int(r[1]) << 64) | (int(r[0]) << 32) | int(r[2]) == comp[j * len(comp) // world]
    # plan: every rank's held range is cut exactly at the shard_ranges boundaries
    for world in (1, 2, 3, 5):
        n = 1000 + world
        all_counts = rng.integers(0, 60, size=(world, world, 8)).astype(np.uint64)
        all_counts[-1, -1, :] += np.uint64(n) - all_counts.sum(axis=(0, 1))  # every layout totals n
        ranges = sharding.shard_ranges(n, world)
        recv = np.zeros((world, 8), dtype=np.uint64)
        for me in range(world):
            cnt, st = sharding.rebalance_plan(all_counts, world, n, me)
            held = all_counts[:, me, :].sum(0)
            assert np.array_equal(cnt.sum(0), held)
            recv += cnt
        for g in range(world):
            assert np.all(recv[g] == ranges[g][1] - ranges[g][0])


def test_ordered_i64_roundtrip_and_order():
    from paper_1712_06326_b200 import sharding
    x = np.array([-np.inf, -1e300, -2.5, -0.0, 0.0, 1e-300, 3.0, np.inf])
    o = sharding.double_to_ordered_i64(x)
    assert np.all(np.diff(o) > 0)
    assert np.array_equal(sharding.ordered_i64_to_double(o).view(np.uint64), x.view(np.uint64))


def test_oracle_fill_loop_with_compiled_reference_knn(golden):
    """The restated run_loop with its k-NN answered by the reference's compiled knn_search (the
    CPU baseline bench.py times) gives the same run as with the linear-scan oracle."""
    tag = "eval_48x40_c_s101_m102"
    img, kn = golden[tag + "__image"], golden[tag + "__known"]
    base = oracle.MultiIndex(img, kn, 9, 0.6, 8)
    out1, r1 = oracle.inpaint(img, kn, 9, 0.6, 8, knn=12, mi=base)
    om = oracle.MultiIndex(img, kn, 9, 0.6, 8)
    om.use_reference_knn(workers=3)
    out2, r2 = oracle.inpaint(img, kn, 9, 0.6, 8, knn=12, mi=om)
    assert len(r1) == len(r2) > 0
    for f in ("tx", "ty", "sx", "sy", "cost", "layout_id", "candidates"):
        assert np.array_equal(r1[f], r2[f]), f
    assert np.array_equal(out1, out2)
    # set_layout round trip: a layout replaced by its own arrays answers identically
    L = base.index(3)
    om2 = oracle.MultiIndex(img, kn, 9, 0.6, 8)
    om2.set_layout(3, L.mean, L.comp, L.lo, L.hi, L.coords, L.keys)
    assert np.array_equal(om2.index(3).coords, L.coords) and np.array_equal(om2.index(3).hi, L.hi)
