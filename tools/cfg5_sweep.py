"""cfg5 sweep (BASELINE.json configs[4]) on one B200.

  python tools/cfg5_sweep.py [--n 20,22,24,26] [--dims 4,8,16] [--queries 65536] [--out FILE]

For every (n, D): n fp32 vectors of dim 125, x = Q diag(0.9^(k/2)) z (seeded, generated on the
device), the vector index built from device memory (PCA fit on the FP64 tensor cores, projection,
quantiser, Morton sort, finalize; CUDA-event time), then 2^16 queries with 40% of their
coordinates unknown:
  * e2e: zi_vector_knn_batch from host memory (queries H2D, make_query, exact k-NN k=80, results
    D2H), wall time;
  * device: the same descriptors through the device-resident batch k-NN (CUDA events), with the
    scanned bytes per query and the HBM fraction (MEASURED_PEAKS.json hbm_gbs).
CPU baseline (n <= 2^22): the reference's compiled knn_search (oracle/_ref, mu=256) on a sample of
the descriptors, queries split over the host threads.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="20,22,24,26")
    ap.add_argument("--dims", default="4,8,16")
    ap.add_argument("--queries", type=int, default=1 << 16)
    ap.add_argument("--k", type=int, default=80)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cfg5_sweep.json"))
    args = ap.parse_args()
    import torch

    import oracle
    import paper_1712_06326_b200 as zb
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    ctx = zb.Context.default()
    dim, k, nq = 125, args.k, args.queries
    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(rng.normal(size=(dim, dim)))
    scale = 0.9 ** (np.arange(dim) / 2.0)
    dev = torch.device("cuda", 0)
    Qt = torch.tensor(Q.T, dtype=torch.float32, device=dev)
    sc = torch.tensor(scale, dtype=torch.float32, device=dev)
    qz = rng.normal(size=(nq, dim)) * scale
    Qh = np.ascontiguousarray((qz @ Q.T).astype(np.float32))
    known = (rng.random((nq, dim)) >= 0.4).astype(np.uint8)
    rows = []
    for ln in (int(x) for x in args.n.split(",")):
        n = 1 << ln
        g = torch.Generator(device=dev).manual_seed(5)
        X = torch.empty((n, dim), dtype=torch.float32, device=dev)
        for b in range(0, n, 1 << 22):
            z = torch.randn((min(1 << 22, n - b), dim), generator=g, dtype=torch.float32, device=dev) * sc
            X[b:b + z.shape[0]] = z @ Qt
        torch.cuda.synchronize()
        for D in (int(x) for x in args.dims.split(",")):
            zb.VectorIndex(X, D, ctx=ctx)  # warm-up
            builds = [zb.VectorIndex(X, D, ctx=ctx).build_ms for _ in range(3)]
            vi = zb.VectorIndex(X, D, ctx=ctx)
            vi.knn(Qh[:512], known[:512], k)
            t0 = time.perf_counter()
            out, cnt = vi.knn(Qh, known, k)
            e2e = time.perf_counter() - t0
            qd = vi.make_queries(Qh, known)
            idx = vi.index()
            ms, stats, _ = idx.knn_batch_bench(qd, k, reps=2)
            P = (D + 3) // 4
            blocks, scored, _ = (int(x) for x in stats)
            alg = scored * (4 * P + 4) + blocks * 8 * P
            row = {"n": n, "D": D, "build_ms": float(np.median(builds)), "build_rows_per_s": n / (np.median(builds) * 1e-3),
                   "e2e_queries_per_s": nq / e2e, "device_queries_per_s": nq / (ms * 1e-3), "device_ms": ms,
                   "scanned_bytes_per_query": alg / nq, "touched_fraction": scored / (nq * n),
                   "achieved_GBps": alg / (ms * 1e-3) / 1e9, "frac_of_hbm": alg / (ms * 1e-3) / 1e9 / hbm,
                   "index_bytes": n * (4 * P + 4)}
            if ln <= 22 and oracle.ref_available():  # the reference's own knn_search on the host
                c, kk = idx.export()
                ref = oracle.RefIndex(c, kk)
                ns = 256 if ln <= 20 else 64
                th = os.cpu_count() or 1
                t0 = time.perf_counter()
                want, _ = ref.knn_batch(qd[:ns], k, threads=th)
                dt = time.perf_counter() - t0
                row["cpu_baseline"] = {"value": ns / dt, "unit": "queries/s", "cores": th, "kind": "reference",
                                       "sample": f"{ns} queries, knn_search (mu=256) over the compiled zcurve_index"}
                row["cpu_equal"] = bool(np.array_equal(want, out[:ns]))
            print(json.dumps(row), flush=True)
            rows.append(row)
            del vi, idx
        del X
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"config": f"cfg5 (BASELINE.json configs[4]): dim 125, 0.9^k eigen-decay, 40 pct unknown query coords, k={k}",
               "queries": nq, "hbm_peak_gbs": hbm, "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
