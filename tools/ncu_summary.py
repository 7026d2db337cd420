"""Summarise ncu --set full reports into profiles/<round>/ text files (dev tool, run here)."""
import csv
import io
import subprocess
import sys

KEYS = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size', 'launch__cluster_dim_x',
        'launch__waves_per_multiprocessor', 'sm__cycles_elapsed.avg.per_second', 'smsp__inst_executed.sum']


def summarize(rep: str, note: str) -> str:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = [note]
    for r in rows[2:]:
        out.append("")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"{k:70s} {units[i]:10s} {r[i]}")
        items = []
        for i, n in enumerate(h):
            if 'smsp__average_warps_issue_stalled' in n and n.endswith('per_issue_active.ratio'):
                try:
                    items.append((float(r[i]), n))
                except ValueError:
                    pass
        out.append("top stall reasons (warps per issue-active cycle):")
        out += [f"   {v:7.3f} {n}" for v, n in sorted(items, reverse=True)[:6]]
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    rep, dst, note = sys.argv[1], sys.argv[2], sys.argv[3]
    open(dst, "w").write(summarize(rep, note))
