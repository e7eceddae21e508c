#!/usr/bin/env python
"""Headline benchmark: 8-layout SFC multi-index build ("dictionary patches indexed/s").
BASELINE.json's metric names no config, so the N=1 line runs the largest single-GPU config:
configs[3] = cfg4 (4096^2 u16-range value noise -> u8, 9x9 patches, D=8, 5% of the 16x16 blocks
removed, n = 14.9 M dictionary patches), synthetic seeded input; cfg2
(configs[1]) and cfg1 stay available through --config.

One step = multi_index::build (proj/src/builder.cpp:202-224) of one image already resident in
HBM: dictionary collection, exact PCA moments (int8 tensor cores), the 8 eigen-solves on the
device, projection + quantisation of all 8 layouts (int8 tensor-core digit GEMM + exact fp64
fix-up), one hybrid Morton sort over the records of all layouts, 8 finalizes.  L2 is flushed
(256 MiB write) before every timed step, outside the timed interval.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config cfg2|cfg1|cfg4]

N > 1 (torchrun): ONE cfg image range-partitioned by Morton key over the ranks (the sharded build
of SURVEY.md §8(e): moments SUM, lo/hi MIN/MAX, sample all-gather, two all-to-alls over NCCL),
strong scaling, timing the max over ranks; --replicas runs one independent image per rank instead
(weak scaling).  --sharded forces the sharded pipeline at N = 1 too (its single-rank overhead).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "dictionary patches indexed/s"
UNIT = "patches/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg4"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-inpaint", action="store_true")
    p.add_argument("--no-knn", action="store_true")
    p.add_argument("--knn-n", type=int, default=1 << 24,
                   help="cfg5-like dictionary size for the k-NN line (2^24 x 20 B = 336 MB > L2: an HBM roofline)")
    p.add_argument("--knn-dims", type=int, default=16)
    p.add_argument("--knn-queries", type=int, default=1 << 14)
    p.add_argument("--no-vector", action="store_true", help="skip the cfg5 vector-index build line")
    p.add_argument("--vec-n", type=int, default=1 << 24, help="cfg5 vector-index rows")
    p.add_argument("--sharded", action="store_true",
                   help="range-partitioned build of ONE image over the N ranks (SURVEY.md §8(e); strong scaling); "
                        "the default when N > 1")
    p.add_argument("--replicas", action="store_true",
                   help="N > 1: one independent image per rank (weak scaling) instead of the sharded build")
    return p.parse_args()


def workload(name: str, rank: int):
    gen = getattr(workloads, name)
    seed = {"cfg1": 1, "cfg2": 2, "cfg4": 4}[name] + 1000 * rank
    img, known, p = gen(seed=seed)
    return img, known, p


# ---------------------------------------------------------------------------- CPU reference arm
def cpu_build_sample(img, known, p, n_sample: int, threads: int):
    """The reference's CPU build on a bounded sample: collect_dictionary (restated) on the whole
    mask, then for the first n_sample dictionary patches the 8 layout builds concurrently
    (multi_index::build with a pool, builder.cpp:212-218): exact moments + Jacobi PCA +
    projection/quantisation (oracle port; Eigen is absent) and the reference's own compiled
    zcurve_index::from_descriptors sort (oracle/_ref) when available."""
    import ctypes as C

    import oracle
    K, D = p["patch_size"], p["dims"]
    ch = 1 if img.ndim == 2 else img.shape[2]
    use_ref = oracle.ref_available()
    R = oracle.ref() if use_ref else None
    t0 = time.perf_counter()
    keys = oracle.collect_dictionary(known, K)[:n_sample]
    n = int(keys.size)
    s, S = oracle.patch_moments(img, K, keys)
    lay = oracle.subset_layouts(K, 0.6)
    dims = min(D, lay.shape[1] * ch, n)

    def one(l):
        cols = oracle.layout_columns(lay[l], K, ch)
        mean, cov = oracle.layout_covariance(s, S, n, cols)
        comp, _ = oracle.pca_from_cov(cov, dims)
        _, _, coords, _ = oracle.project_build(img, keys, lay[l], mean, comp)
        if R is not None:
            h = R.zr_index_create(coords.ctypes.data_as(C.POINTER(C.c_uint8)),
                                  keys.ctypes.data_as(C.POINTER(C.c_uint32)), n, dims)
            R.zr_index_free(h)
        else:
            oracle.from_descriptors(coords, keys)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, range(8)))
    dt = time.perf_counter() - t0
    kind = "reference" if use_ref else "port"
    sample = (f"{n} of the dictionary patches of {img.shape[1]}x{img.shape[0]}x{ch} "
              f"({'K=%d D=%d' % (K, dims)}), all 8 layouts on {threads} threads; sort = "
              f"{'the reference zcurve.cpp compiled from source' if use_ref else 'oracle port'}, "
              f"PCA/projection = oracle port (Eigen absent)")
    return n / dt, dt, kind, sample


BUILD_SAMPLE = {"cfg1": 58368, "cfg2": 131072, "cfg4": 262144}


def cpu_inpaint_baseline(mi, img, known, p, max_iter: int):
    """The reference's fill loop on the host: the restated run_loop (engine.cpp:371-438; priorities,
    std::set order, make_query, masked-cost refine, paste) whose k-NN queries go to the reference's
    OWN compiled knn_search (zcurve.cpp:429-452) over its own zcurve_index per layout, on a
    priority_pool of nproc - 1 threads (run_loop's default workers = cores, engine.cpp:454-458).
    The 8 indices are the device build's (bit-identical to the reference's, tests/test_gpu_scale.py),
    re-sorted by the compiled from_descriptors; timed over the first max_iter iterations."""
    import oracle
    K, D = p["patch_size"], mi.dims
    pm = np.stack([mi.layout(l)["mean"] for l in range(8)])
    pc = np.stack([mi.layout(l)["components"] for l in range(8)])
    om = oracle.MultiIndex(img, known, K, 0.6, D, pca_mean=pm, pca_comp=pc, layouts=[])
    for l in range(8):
        lay = mi.layout(l)
        c, k = mi.index_arrays(l)
        om.set_layout(l, lay["mean"], lay["components"], lay["lo"], lay["hi"], c, k)
    workers = om.use_reference_knn()
    t0 = time.perf_counter()
    _, recs = oracle.inpaint(img, known, K, 0.6, D, knn=p["knn"], mi=om, max_iter=max_iter)
    dt = time.perf_counter() - t0
    return {"value": len(recs) / dt, "unit": "iterations/s", "cores": workers, "kind": "reference",
            "seconds": dt, "iterations": int(len(recs)),
            "sample": f"the first {len(recs)} fill-loop iterations of this config; query = the reference's compiled "
                      f"knn_search (mu=256, nu=2048) on priority_pool({workers - 1}), fill loop / make_query / refine "
                      f"= oracle restatement of engine.cpp (Eigen absent)"}


def cpu_brute_baseline(img, targets, keys, K, n_queries: int = 2):
    """The reference's brute_force_best (engine.cpp:220-236) is single-threaded: the restated scan
    over the whole dictionary, timed on the first n_queries targets."""
    import oracle
    t0 = time.perf_counter()
    for tv, tk in targets[:n_queries]:
        oracle.brute_force_best(img, tv, tk, K, keys)
    dt = (time.perf_counter() - t0) / n_queries
    return {"value": 1.0 / dt, "unit": "queries/s", "cores": 1, "kind": "port", "us_per_query": dt * 1e6,
            "sample": f"{n_queries} of the {len(targets)} targets, whole dictionary ({keys.size} patches), "
                      f"restated single-thread brute_force_best"}


def run_reference(args, rank):
    if rank != 0:
        return
    img, known, p = workload(args.config, 0)
    threads = max(1, min(8, os.cpu_count() or 1))
    n_sample = BUILD_SAMPLE[args.config]
    for _ in range(args.warmup):
        cpu_build_sample(img, known, p, n_sample, threads)
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        v, dt, kind, sample = cpu_build_sample(img, known, p, n_sample, threads)
        vals.append(dt)
    total = time.perf_counter() - t_all
    value = n_sample * args.steps / sum(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u8",
            "data": "synthetic", "config": {"workload": f"{args.config}: bounded sample of its dictionary "
                                                        f"({n_sample} patches x 8 layouts per step)",
                                            "parallelism": f"cpu threads x{threads} (one per layout, "
                                                           f"multi_index::build's pool)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.lines = []
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        self.mark = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def begin(self):
        self.mark = time.perf_counter()

    def end(self):
        self.stop_t = time.perf_counter()

    def result(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        rows = [l for t, l in self.lines if self.mark is not None and self.mark - 0.15 <= t <= self.stop_t + 0.15]
        if not rows:
            rows = [l for _, l in self.lines[-3:]]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- roofline model
def pt_groups(D: int):
    """Layout groups of the int8 tensor-core projection (k_proj_tc.cu): five digit columns per
    (layout, dim), at most 256 MMA columns per group (padded to a multiple of 16), the layouts
    spread evenly over the fewest groups."""
    nlmax = min(8, 256 // (5 * D))
    ng = (8 + nlmax - 1) // nlmax
    nlmax = (8 + ng - 1) // ng
    out, l0 = [], 0
    while l0 < 8:
        nl = min(nlmax, 8 - l0)
        out.append((nl, (nl * 5 * D + 15) // 16 * 16))
        l0 += nl
    return out


def pt_launches(D: int) -> int:
    """Projection launches per pass: one per layout group, or a single launch when the two groups
    of four layouts of D = 7..10 are fed from one gathered tile (k_proj_tc.cu, pt_plan::fuse)."""
    gs = pt_groups(D)
    if len(gs) == 2 and gs[0] == gs[1] and gs[0][0] == 4 and 7 <= D <= 10 and not os.environ.get("ZI_PROJ_NOFUSE"):
        return 1
    return len(gs)


def algorithmic_bytes(kernel: str, n: int, D: int, mc: int, F: int = 0) -> float | None:
    """Algorithmic HBM bytes per launch; gathered pixels are L1/L2 served.
    The radix passes and the window sort run once over the records of all 8 layouts (N = 8n);
    the tensor-core projection launches once per (pass, layout group) -- once per pass when the
    groups share a gathered tile (pt_launches): keys in, and in the quantise pass the Morton
    records of its layouts out (averaged over the launches)."""
    W = (D + 3) // 4
    N = 8 * n
    g = pt_launches(D) if D <= 16 else 1
    return {
        "radix_onesweep": 2 * 4 * (W + 1) * N,          # legacy LSD sort: read + write of (W key words + payload)
        "segment_sort": 2 * 4 * (W + 1) * N,            # one read + one in-place write per record
        "ssort_count": 4 * (W + 1) * N,                 # splitter sort: records read, bucket histograms
        "ssort_scatter": 2 * 4 * (W + 1) * N,           # records read + written to their buckets
        "ssort_local": 2 * 4 * (W + 1) * N,             # every bucket read + written back in order
        "radix_hist": 4 * (W + 1) * N,
        "radix_count": 4 * N,                           # the digit word of every record (tile counts: ~0.3 %)
        "index_bbox": 4 * W * N,                        # fused final pass: the 8 indices' dim planes read once
        "proj_minmax": 8 * D * n,
        "quantize_interleave": (8 * D + 4 + 4 * (W + 1)) * n,
        "finalize_index": (4 * (W + 1) + 4 * (W + 1)) * n,
        "project_tc_minmax": 4 * n,
        "project_tc_quantize": (4 * n * g + 4 * (W + 1) * N) / g,
    }.get(kernel)


def algorithmic_ops(kernel: str, n: int, D: int, mc: int, F: int = 0) -> float | None:
    """Tensor-core ops per launch: the fp64 projection (2 per FMA over the layout's m*C columns),
    or the int8 digit GEMM of the tensor-core projection (2 * n * Fpad * columns, averaged over
    its launches)."""
    if kernel == "project":
        return 2.0 * n * mc * D
    if kernel in ("project_tc_minmax", "project_tc_quantize") and D <= 16:
        Fpad = (F + 127) // 128 * 128
        gs = pt_groups(D)
        return 2.0 * n * Fpad * sum(npad for _, npad in gs) / pt_launches(D)
    return None


# B200 FP64 tensor-core peak: not in MEASURED_PEAKS.json (driver measures bf16 only) nor in the
# profiling recipe -> NVIDIA's B200 datasheet figure.  The int8 dense tensor rate is twice the bf16
# rate on B200 (datasheet 4.5 POPS vs 2.25 PFLOPS): 2 x the measured bf16 burst.
FP64_TENSOR_PEAK_TFLOPS = 40.0


def tensor_peak(kernel: str, peaks: dict):
    if kernel.startswith("project_tc"):
        bf = float(peaks.get("bf16_tflops", 2250.0))
        return 2.0 * bf, "2 x MEASURED_PEAKS.json bf16_tflops (int8 = 2x bf16 dense on B200)", "s8/u8 -> s32 (tcgen05.mma kind::i8)"
    return FP64_TENSOR_PEAK_TFLOPS, "B200 datasheet FP64 Tensor Core 40 TFLOPS (no measured fp64 peak)", "f64 (mma.m8n8k4.f64)"


def vector_index_line(zb, ctx, args):
    """cfg5 (BASELINE configs[4]) on the device end to end: PCA fit of n fp32 vectors of dim 125
    (canonical-order mean / covariance on the FP64 tensor cores + device eigen-solve),
    projection, quantiser, Morton sort; then 2^14 queries with 40% unknown coordinates through
    make_query + exact k-NN.  Rows are generated on the device (seeded torch normals) and are
    resident in HBM when the timed build starts."""
    import torch
    n, dim, D, nq, k = args.vec_n, 125, 16, 1 << 14, 80
    dev = torch.device("cuda", torch.cuda.current_device())
    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(rng.normal(size=(dim, dim)))
    scale = torch.tensor(0.9 ** (np.arange(dim) / 2.0), dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev).manual_seed(5)
    X = torch.empty((n, dim), dtype=torch.float32, device=dev)
    Qt = torch.tensor(Q.T, dtype=torch.float32, device=dev)
    for b in range(0, n, 1 << 22):
        z = torch.randn((min(1 << 22, n - b), dim), generator=g, dtype=torch.float32, device=dev) * scale
        X[b:b + z.shape[0]] = z @ Qt
    torch.cuda.synchronize()
    zb.VectorIndex(X, D, ctx=ctx)  # warm-up (pool, module load)
    ctx.set_profiling(True)
    times = []
    for _ in range(3):
        vi = zb.VectorIndex(X, D, ctx=ctx)
        times.append(vi.build_ms)
    prof = ctx.profile()
    ctx.set_profiling(False)
    build_ms = float(np.median(times))
    qz = rng.normal(size=(nq, dim)) * (0.9 ** (np.arange(dim) / 2.0))
    Qh = (qz @ Q.T).astype(np.float32)
    known = (rng.random((nq, dim)) >= 0.4).astype(np.uint8)
    vi.knn(Qh[:256], known[:256], k)
    t0 = time.perf_counter()
    out, cnt = vi.knn(Qh, known, k)
    qdt = time.perf_counter() - t0
    return {"workload": f"cfg5: n={n} fp32 vectors, dim {dim}, D={D} (x = Q diag(0.9^(k/2)) z, seeded), "
                        f"{nq} queries with 40% unknown coordinates, k={k}, L2",
            "build_ms": build_ms, "rows_per_s": n / (build_ms * 1e-3), "build_ms_all": times,
            "build_kernels_ms": {kk: v[0] / 3 for kk, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
            "query_e2e_queries_per_s": nq / qdt, "query_e2e_s": qdt,
            "note": "X resident in HBM (device-generated); queries through zi_vector_knn_batch from host memory "
                    "(H2D, make_query, k-NN, D2H inside the timing)"}


def candidate_scoring(zb, ctx, args, hbm_peak):
    """cfg5-style batched k-NN (the reference's Python knn_search path over u8 descriptors):
    dictionary sorted on the device, then nq queries answered by the warp-per-query kernel."""
    import oracle
    n, D, nq, k = args.knn_n, args.knn_dims, args.knn_queries, 80
    coords, queries = workloads.cfg5_descriptors(n, D, nq)
    keys = np.arange(n, dtype=np.uint32)
    ctx.synchronize()
    ctx.timer_start()
    idx = zb.ZCurveIndex.from_descriptors(coords, keys, D, ctx=ctx)
    sort_ms = ctx.timer_stop()
    ms, stats, _ = idx.knn_batch_bench(queries, k, reps=3)
    P = (D + 3) // 4
    blocks, scored, results = (int(x) for x in stats)
    alg = scored * (4 * P + 4) + blocks * 8 * P
    full = n * (4 * P + 4) + (n // 256) * 8 * P
    line = {"workload": f"cfg5-like: n={n} u8 descriptors D={D} (top-D PCA coords of 0.9^k-decay Gaussians), "
                        f"{nq} queries with 40% of 125 coords unknown, k={k}, L2",
            "queries_per_s": nq / (ms * 1e-3), "ms_per_batch": ms,
            "algorithmic_bytes_per_query": alg / nq, "full_scan_bytes_per_query": full,
            "touched_fraction": scored / (nq * n),
            "achieved_GBps": alg / (ms * 1e-3) / 1e9, "frac_of_hbm": alg / (ms * 1e-3) / 1e9 / hbm_peak,
            "index_bytes": n * (4 * P + 4), "from_descriptors_ms_incl_h2d": sort_ms,
            "note": "index bytes vs the 126 MB L2 decide whether this is an HBM or an L2 roofline"}
    # CPU: the reference's own knn_search (compiled zcurve.cpp), sequential, on a query sample
    if oracle.ref_available():
        import ctypes as C
        R = oracle.ref()
        sc, sk = idx.export()
        h = R.zr_index_create(sc.ctypes.data_as(C.POINTER(C.c_uint8)), sk.ctypes.data_as(C.POINTER(C.c_uint32)), n, D)
        ns = 32
        out = np.zeros(ns * k, dtype=np.uint64)
        qs = np.ascontiguousarray(queries[:ns])
        t0 = time.perf_counter()
        R.zr_index_knn_batch(h, qs.ctypes.data_as(C.POINTER(C.c_uint8)), ns, k, 256, 2048, 0, 1,
                             out.ctypes.data_as(C.POINTER(C.c_uint64)))
        dt = time.perf_counter() - t0
        R.zr_index_free(h)
        line["cpu_baseline"] = {"value": ns / dt, "unit": "queries/s", "cores": 1, "kind": "reference",
                                "sample": f"first {ns} queries, sequential knn_search (mu=256)"}
    return line


def run_sharded(args, zb, world, rank, local, dist):
    """One image (seed of rank 0) range-partitioned over the ranks: every step
    is the whole sharded build from the device-resident image (dictionary, moments SUM over NCCL,
    8 PCA models, lo/hi MIN/MAX, projection + quantiser, local sort, sample all-gather, two
    all-to-alls, finalize), timed on the ctx stream; the step time is the max over ranks and the
    value counts the image's dictionary once (strong scaling).  e2e: the same build from host
    memory through a fresh shard (image + mask upload inside the timing)."""
    from paper_1712_06326_b200 import sharding
    img, known, p = workload(args.config, 0)
    ctx = zb.Context(local)
    cfg = zb.index_config(patch_size=p["patch_size"], dims=p["dims"], knn=p["knn"])
    if dist is not None:
        import torch
        comm = sharding.TorchComm(device=torch.device("cuda", local))
    else:
        comm = sharding.LoopbackComm(1)
    sh = sharding.DeviceShard(img, known, cfg, rank, world, ctx=ctx)
    info = sharding.build_sharded([sh], comm)

    def build():
        sh.rebuild()
        return sharding.build_sharded([sh], comm)

    for _ in range(max(args.warmup, 0)):
        build()
    ctx.synchronize()
    clocks = ClockSampler(local)
    launches0 = ctx.kernel_launches
    if dist is not None:
        dist.barrier()
    clocks.begin()
    total_ms = 0.0
    for _ in range(args.steps):
        ctx.flush_l2()
        ctx.timer_start()
        info = build()
        total_ms += ctx.timer_stop()
    clocks.end()
    launches = ctx.kernel_launches - launches0
    n_total = sh.n_total
    e2e_ms = 0.0
    for _ in range(max(1, args.steps // 4)):
        ctx.synchronize()
        ctx.timer_start()
        fresh = sharding.DeviceShard(img, known, cfg, rank, world, ctx=ctx)
        sharding.build_sharded([fresh], comm)
        e2e_ms += ctx.timer_stop()
        del fresh
    e2e_steps = max(1, args.steps // 4)
    if dist is not None:
        import torch
        t = torch.tensor([total_ms, e2e_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0].item()), float(t[1].item())
    value = n_total * args.steps / (total_ms * 1e-3)
    if rank == 0:
        h2d = img.nbytes + known.nbytes
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u8+i8+f64", "data": "synthetic",
                "config": {"workload": f"{args.config}: one image range-partitioned by Morton key over {world} rank(s), "
                                       f"n={n_total} dictionary patches, 8 layout indices",
                           "global_batch": n_total, "parallelism": f"range-partitioned x{world} (sample sort over NCCL)",
                           "l2": "flushed (256 MiB write) before every timed step"},
                "e2e": {"value": n_total * e2e_steps / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": 0, "ms_per_step": e2e_ms / e2e_steps,
                        "api": "sharding.DeviceShard (host image + mask in) + build_sharded (zi_shard_*)"},
                "exchange": info, "gpu_launches": launches, "clocks": clocks.result()}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist

    import paper_1712_06326_b200 as zb
    if args.sharded or (world > 1 and not args.replicas):
        run_sharded(args, zb, world, rank, local, dist)
        return

    img, known, p = workload(args.config, rank)
    ctx = zb.Context(local)
    cfg = zb.index_config(patch_size=p["patch_size"], dims=p["dims"], knn=p["knn"])
    clocks = ClockSampler(local)
    mi = zb.MultiIndex(img, known, cfg, ctx=ctx)
    n = mi.n
    for _ in range(max(args.warmup, 0)):
        mi.rebuild()
    ctx.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    # -------- one profiled build outside the timed region: every kernel's launches and device time
    # (the breakdown and the step's algorithmic bytes); timing all ~40 launches costs ~8 % of the
    # step in event records, so the timed region below times only the step's largest kernels
    ctx.flush_l2()
    ctx.set_profile_filter(None)
    ctx.set_profiling(True)
    mi.rebuild()
    ctx.synchronize()
    prof_all = ctx.profile()
    ctx.set_profiling(False)
    timed_kernels = [k for k, _ in sorted(prof_all.items(), key=lambda kv: -kv[1][0])[:4]]

    # -------- timed region: K builds from the HBM-resident image
    ctx.set_profile_filter(timed_kernels)
    ctx.set_profiling(True)
    launches0 = ctx.kernel_launches
    barrier()
    ctx.synchronize()
    clocks.begin()
    step_ms = []
    host_eigen = []
    for _ in range(args.steps):
        ctx.flush_l2()
        ctx.timer_start()
        mi.rebuild()
        step_ms.append(ctx.timer_stop())
        host_eigen.append(mi.info.eigen_seconds)
    ctx.synchronize()
    clocks.end()
    barrier()
    launches = ctx.kernel_launches - launches0
    prof = ctx.profile()
    ctx.set_profiling(False)
    ctx.set_profile_filter(None)
    total_ms = sum(step_ms)
    n_total = n
    if dist is not None:
        import torch
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        c = torch.tensor([n], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        n_total = int(c.item())
    value = n_total * args.steps / (total_ms * 1e-3)

    # -------- roofline of the dominant kernel (live CUDA-event durations over the timed region)
    mc = mi.m * mi.channels
    breakdown = {k: {"ms_per_step": v[0], "launches_per_step": v[1]}
                 for k, v in sorted(prof_all.items(), key=lambda kv: -kv[1][0])}
    # kernels timed in the region (>0 launches); with the splitter sort the onesweep passes only
    # sort its ~N/70 samples, so their per-N byte count does not apply
    prof = {k: v for k, v in prof.items() if v[1] > 0 and v[0] > 0}
    if "ssort_local" in prof_all:
        prof.pop("radix_onesweep", None)
        prof_all = {k: v for k, v in prof_all.items() if k != "radix_onesweep" or v[1] == 0}
    dom = max(prof.items(), key=lambda kv: kv[1][0]) if prof else None
    roofline = None
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic_db = {}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic_db = json.load(f)
    except OSError:
        pass
    # roofline of the dominant tensor-core kernel of the step (the projection) and, beside it, of
    # the dominant HBM-bound kernel
    def hbm_roofline(kname, kms, kl):
        per_launch_ms = kms / max(kl, 1)
        b = algorithmic_bytes(kname, n, mi.dims, mc, F)
        achieved = b / (per_launch_ms * 1e-3) / 1e9
        tr = traffic_db.get(args.config, {}).get(kname)
        return {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": tr, "bytes_per_launch": b,
                "avg_launch_ms": per_launch_ms,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650"}

    F = p["patch_size"] ** 2 * (1 if img.ndim == 2 else img.shape[2])
    Fpad = (F + 127) // 128 * 128
    hbm_kernels = {k: v for k, v in prof.items() if algorithmic_ops(k, n, mi.dims, mc, F) is None
                   and algorithmic_bytes(k, n, mi.dims, mc, F) is not None}
    roofline_hbm = None
    if hbm_kernels:
        kname, (kms, kl) = max(hbm_kernels.items(), key=lambda kv: kv[1][0])
        roofline_hbm = hbm_roofline(kname, kms, kl)
    tensor_kernels = {k: v for k, v in prof.items() if algorithmic_ops(k, n, mi.dims, mc, F) is not None}
    if tensor_kernels and (dom is None or dom[0] in tensor_kernels or dom[0] not in hbm_kernels):
        kname, (kms, kl) = max(tensor_kernels.items(), key=lambda kv: kv[1][0])
        per_launch_ms = kms / max(kl, 1)
        fl = algorithmic_ops(kname, n, mi.dims, mc, F)
        achieved = fl / (per_launch_ms * 1e-3) / 1e12
        peak, src, dt = tensor_peak(kname, peaks)
        roofline = {"kernel": kname, "bound": "tensor", "achieved": achieved, "peak": peak,
                    "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": traffic_db.get(args.config, {}).get(kname), "ops_per_launch": fl,
                    "avg_launch_ms": per_launch_ms, "dtype": dt, "peak_source": src,
                    "note": "int8 digit GEMM (five balanced base-256 digits of the fp64 components) with the "
                            "exact fp64 fix-up; the epilogue (integer min/max, bracket quantisation, Morton "
                            "interleave) bounds it, not the MMA" if kname.startswith("project_tc") else
                            "D=12 fills 12 of the 16 MMA columns, so the useful-flop ceiling is 0.75 of peak"}
    else:
        roofline = roofline_hbm

    # whole-step floor: max(HBM bytes / BW, tensor ops / tensor peak) with this pipeline's own
    # algorithmic bytes (every counted kernel, per step)
    extra = {"project": (4 + 8 * mi.dims) * n,        # dictionary keys in, fp64 projections out
             "patch_matrix": (4 + Fpad) * n,            # keys in, feature-major patch matrix out
             "patch_moments": Fpad * n}                 # the patch matrix read once
    def step_b(k):
        b = algorithmic_bytes(k, n, mi.dims, mc, F)
        return b if b is not None else extra.get(k)
    step_bytes = sum(step_b(k) * v[1] for k, v in prof_all.items() if step_b(k) is not None)
    step_t = 0.0
    for k, v in prof_all.items():
        o = algorithmic_ops(k, n, mi.dims, mc, F)
        if o is not None:
            step_t += o * v[1] / (tensor_peak(k, peaks)[0] * 1e12)
    floor_ms = max(step_bytes / (hbm_peak * 1e9), step_t) * 1e3
    step_roofline = {"floor_ms": floor_ms, "measured_ms": total_ms / args.steps,
                     "frac": floor_ms / (total_ms / args.steps), "hbm_bytes_per_step": step_bytes,
                     "tensor_ms_per_step": step_t * 1e3,
                     "binding": "tensor" if step_t > step_bytes / (hbm_peak * 1e9) else "hbm"}

    # -------- e2e through the public C ABI with pinned host buffers
    e2e = None
    try:
        import torch
        pin_img = torch.from_numpy(np.ascontiguousarray(img)).pin_memory()
        pin_known = torch.from_numpy(np.ascontiguousarray(known)).pin_memory()
        pin_keys = torch.empty(n, dtype=torch.int32).pin_memory()
        ptr_img = zb._lib.C.cast(pin_img.data_ptr(), zb._lib.u8p)
        ptr_known = zb._lib.C.cast(pin_known.data_ptr(), zb._lib.u8p)
        ptr_keys = zb._lib.C.cast(pin_keys.data_ptr(), zb._lib.u32p)
        L = zb._lib.lib()
        h, w = known.shape
        ch = 1 if img.ndim == 2 else img.shape[2]
        e2e_ms = []
        for it in range(args.warmup + args.steps):
            ctx.synchronize()
            ctx.timer_start()
            hmi = zb._lib.C.c_void_p()
            nd = zb._lib.C.c_uint64(0)
            zb._lib.check(L.zi_multi_index_build_to(ctx.h, ptr_img, ptr_known, w, h, ch, zb._lib.C.byref(cfg),
                                                    ptr_keys, n, zb._lib.C.byref(nd), zb._lib.C.byref(hmi)))
            ms = ctx.timer_stop()
            if nd.value != n:
                raise RuntimeError(f"build_to: {nd.value} dictionary keys, expected {n}")
            zb._lib.check(L.zi_multi_index_destroy(hmi))
            if it >= args.warmup:
                e2e_ms.append(ms)
        e2e_total = sum(e2e_ms)
        if dist is not None:
            t = torch.tensor([e2e_total], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_total = float(t.item())
        e2e = {"value": n_total * args.steps / (e2e_total * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(img.nbytes + known.nbytes), "d2h_bytes_per_step": int(4 * n),
               "ms_per_step": e2e_total / args.steps,
               "api": "zi_multi_index_build_to: image + mask H2D, the 8-layout build and the dictionary D2H in one "
                      "call (pinned host buffers; the copies run on the copy engines beside the kernels)"}
    except Exception as ex:  # noqa: BLE001
        e2e = {"error": repr(ex)}

    clk = clocks.result()

    # -------- the fill loop on the built index (inpaint iterations/s), rank 0
    inpaint = None
    if rank == 0 and not args.no_inpaint:
        dt = None
        for _ in range(2):  # timed without per-launch profiling events; the faster of two runs
            t0 = time.perf_counter()
            _, recs, st = mi.inpaint()
            t1 = time.perf_counter() - t0
            dt = t1 if dt is None or t1 < dt else dt
        ctx.set_profiling(True)  # second run: device time per launch
        mi.inpaint()
        kp = ctx.profile()
        ctx.set_profiling(False)
        it = max(int(st.iterations), 1)
        inpaint = {"iterations": int(st.iterations), "seconds": dt, "iterations_per_s": st.iterations / dt,
                   "first_2000_iterations_per_s": min(2000, len(recs)) / float(np.sum(recs["elapsed_seconds"][:2000])),
                   "unit": "iterations/s", "mean_iteration_us": 1e6 * float(np.mean(recs["elapsed_seconds"])),
                   "device_us_per_iteration": {k: 1e3 * v[0] / it for k, v in kp.items()},
                   "note": "sequential fill loop over the built index (host priorities + one device query "
                           "per iteration), through MultiIndex.inpaint / zi_inpaint_with_index; the faster of "
                           "two runs (the host part varies by ~15 % between runs); first_2000_iterations_per_s sums "
                           "the per-iteration wall times of the first 2000 (the CPU baseline's sample)"}
        if world == 1 and not args.no_cpu_baseline:
            try:
                inpaint["cpu_baseline"] = cpu_inpaint_baseline(mi, img, known, p, 2000)
            except Exception as ex:  # noqa: BLE001
                inpaint["cpu_baseline"] = {"error": repr(ex)}

    # -------- the exhaustive masked-L2 scan (brute_force_best, the original method's comparison
    # path, proj/src/engine.cpp:220-236) over the whole dictionary, rank 0
    brute = None
    if rank == 0 and not args.no_inpaint:
        ys, xs = np.nonzero(known == 0)
        K = p["patch_size"]
        pick = np.linspace(0, len(xs) - 1, 16).astype(int)
        targets = []
        for t in pick:  # windows centred on unknown pixels near known ones (fill-front-like)
            x0, y0 = int(xs[t]) - K // 2, int(ys[t]) - K // 2
            tv = np.zeros((K, K) + img.shape[2:], np.uint8)
            tk = np.zeros((K, K), np.uint8)
            for r in range(K):
                for c in range(K):
                    yy, xx = y0 + r, x0 + c
                    if 0 <= yy < img.shape[0] and 0 <= xx < img.shape[1] and known[yy, xx]:
                        tv[r, c] = img[yy, xx]
                        tk[r, c] = 1
            targets.append((tv.reshape(-1), tk.reshape(-1)))
        mi.brute_force_best(*targets[0])  # warm-up
        t0 = time.perf_counter()
        for tv, tk in targets:
            mi.brute_force_best(tv, tk)
        dt = (time.perf_counter() - t0) / len(targets)
        ctx.set_profile_filter(["brute_force"])  # device time of the scan kernel alone
        ctx.set_profiling(True)
        for tv, tk in targets:
            mi.brute_force_best(tv, tk)
        bp = ctx.profile().get("brute_force", (0.0, 1))
        ctx.set_profiling(False)
        ctx.set_profile_filter(None)
        dev_dt = bp[0] * 1e-3 / max(bp[1], 1)
        C = 1 if img.ndim == 2 else img.shape[2]
        known_vals = float(np.mean([int(tk.sum()) for _, tk in targets])) * C
        ops = 3.0 * n * known_vals  # subtract, square (multiply-add) per known value, per dictionary patch
        int_peak = 148 * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12  # TOPS, nominal INT32 rate
        brute = {"queries_per_s": 1.0 / dt, "us_per_query": dt * 1e6, "device_us_per_query": dev_dt * 1e6,
                 "dictionary": n, "mean_known_values": known_vals, "int_ops_per_query": ops,
                 "achieved_TOPS": ops / dev_dt / 1e12, "int32_peak_TOPS": int_peak,
                 "frac_of_int32": ops / dev_dt / 1e12 / int_peak,
                 "note": "queries_per_s / us_per_query: host wall time per zi_brute_force_best call (target H2D, "
                         "one scan kernel, winner D2H); achieved_TOPS from the kernel's own CUDA-event time. "
                         "INT-compute-bound, not an HBM roofline (SURVEY.md §8(d))"}
        if world == 1 and not args.no_cpu_baseline:
            try:
                brute["cpu_baseline"] = cpu_brute_baseline(img, targets, mi.dictionary, K)
            except Exception as ex:  # noqa: BLE001
                brute["cpu_baseline"] = {"error": repr(ex)}

    knn = None
    if rank == 0 and not args.no_knn:
        try:
            knn = candidate_scoring(zb, ctx, args, hbm_peak)
        except Exception as ex:  # noqa: BLE001
            knn = {"error": repr(ex)}

    vec = None
    if rank == 0 and not args.no_vector:
        try:
            vec = vector_index_line(zb, ctx, args)
        except Exception as ex:  # noqa: BLE001
            vec = {"error": repr(ex)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = max(1, min(8, os.cpu_count() or 1))
            v, dt, kind, sample = cpu_build_sample(img, known, p, min(BUILD_SAMPLE[args.config], n), threads)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample, "seconds": dt}
        except Exception as ex:  # noqa: BLE001
            cpu = {"error": repr(ex)}

    if rank == 0:
        ch = 1 if img.ndim == 2 else img.shape[2]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8+f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {img.shape[1]}x{img.shape[0]}x{ch} u8, K={p['patch_size']}, "
                                   f"D={mi.dims}, 8 layout indices, n={n} dictionary patches per rank",
                       "global_batch": n_total, "parallelism": f"replicas x{world} (independent images)",
                       "l2": "flushed (256 MiB write) before every timed step"},
            "roofline": roofline, "roofline_hbm": roofline_hbm, "step_roofline": step_roofline,
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk, "inpaint": inpaint, "brute_force": brute, "candidate_scoring": knn, "vector_index": vec,
            "breakdown": {"host_eigen_s_per_step": float(np.mean(host_eigen)), "kernels": breakdown},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
