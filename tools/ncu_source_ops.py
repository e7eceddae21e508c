"""Dev: per-opcode and per-position stall samples / shared-memory wavefronts from an
`ncu --page source --csv --print-source sass` dump.  Usage: ncu_source_ops.py dump.csv [kernel#]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
heads = [i for i, r in enumerate(rows) if r and r[0] == 'Address']
start = heads[which]
end = heads[which + 1] if which + 1 < len(heads) else len(rows)
h = rows[start]
seg = [r for r in rows[start + 1:end] if len(r) == len(h)]
iS, iSrc, iW, iWI, iE = (h.index(k) for k in ('# Samples', 'Source', 'L1 Wavefronts Shared', 'L1 Wavefronts Shared Ideal', 'Instructions Executed'))


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def opc(src):
    t = src.split()
    op = t[1] if t[0].startswith('@') else t[0]
    return op.split('.')[0]


tot = sum(f(r[iS]) for r in seg) or 1
print("samples", tot, "instructions", len(seg))
agg, wf, wfi, ex = (collections.Counter() for _ in range(4))
for r in seg:
    op = opc(r[iSrc])
    agg[op] += f(r[iS]); wf[op] += f(r[iW]); wfi[op] += f(r[iWI]); ex[op] += f(r[iE])
for op, v in agg.most_common(20):
    print(f"{op:10s} samples {100 * v / tot:5.1f}%  exec {ex[op]:12.0f} smem_wf {wf[op]:12.0f} ideal {wfi[op]:12.0f}")
print("total smem wavefronts", sum(wf.values()), "ideal", sum(wfi.values()), "instr", sum(ex.values()))
for b in range(0, len(seg), 60):
    s = sum(f(r[iS]) for r in seg[b:b + 60])
    ops = collections.Counter(opc(r[iSrc]) for r in seg[b:b + 60])
    print(b, f"{100 * s / tot:5.1f}%", ops.most_common(5))
