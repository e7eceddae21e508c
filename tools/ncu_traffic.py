"""Per-kernel DRAM traffic and time from an ncu --set full report -> profiles/traffic.json entry.

  python tools/ncu_traffic.py REPORT.ncu-rep CONFIG [--out profiles/traffic.json]

traffic = dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over the captured
launches of each kernel), keyed by bench.py's launch names.
"""
import csv
import io
import json
import os
import subprocess
import sys

NAMES = {"k_onesweep": "radix_onesweep", "k_sort_hist": "radix_hist", "k_lsd_count": "radix_count",
         "k_lsd_chunk_sum": "radix_scan", "k_lsd_chunk_scan": "radix_scan", "k_lsd_offsets": "radix_scan",
         "k_brute8": "brute_force", "k_proj_tc": None, "k_finalize": "finalize_index",
         "k_query_lat": "query_one", "k_brute4": "brute_force", "k_brute": "brute_force", "k_segsort": "segment_sort",
         "k_gram_fused": "patch_moments_fused", "k_vec_gram_blk": "vec_gram", "k_vec_project": "vec_project",
         "k_knn_batch": "knn_batch"}


def main():
    rep, cfg = sys.argv[1], sys.argv[2]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    acc = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        base = name.split("(")[0].split("<")[0].split()[-1]
        key = NAMES.get(base, base)
        if base == "k_proj_tc":  # template arg MODE: 0 = min/max pass, 1 = quantise pass
            key = "project_tc_minmax" if "0," in name.split("<", 1)[1][:12].replace(" ", "") else "project_tc_quantize"
        b = float(r[h.index("dram__bytes_read.sum")]) + float(r[h.index("dram__bytes_write.sum")])
        unit_r = rows[1][h.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit_r, 1)
        t = float(r[h.index("gpu__time_duration.sum")])
        acc.setdefault(key, []).append((b * scale, t))
    db = json.load(open(out)) if os.path.exists(out) else {}
    ent = {k: sum(b for b, _ in v) / len(v) for k, v in acc.items()}
    ent["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over the launches) from one "
                    f"ncu --set full capture ({os.path.basename(rep)}); cold-cache replay, clocks uncontrolled")
    db[cfg] = ent
    json.dump(db, open(out, "w"), indent=1)
    for k, v in sorted(ent.items()):
        print(k, v)


if __name__ == "__main__":
    main()
