"""Summarise ncu --set full reports (raw page) -- dev tool."""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum', 'launch__grid_size']


def summary(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    units = rows[1]
    lines = []
    for r in rows[2:]:
        lines.append(f"== {r[h.index('Kernel Name')][:60]}")
        st = []
        for i, nm in enumerate(h):
            if nm.startswith('smsp__pcsamp_warps_issue_stalled') and not nm.endswith('not_issued'):
                try:
                    st.append((float(r[i]), nm.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        lines.append("   stalls: " + ", ".join(f"{n}={100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:7]))
        for k in KEYS:
            if k in h:
                lines.append(f"   {k} = {r[h.index(k)]} {units[h.index(k)]}")
    return "\n".join(lines)


if __name__ == '__main__':
    for p in sys.argv[1:]:
        print(summary(p))
