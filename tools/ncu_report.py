"""Markdown summary of one ncu capture: raw metrics (--page raw --csv) and the
pc-sampling stall mix (--page source --csv --print-source sass)."""
import collections
import csv
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
           "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "l1tex__t_sector_hit_rate.pct",
           "lts__t_sector_hit_rate.pct"]


def raw_table(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    out = [f"## `{name[:110]}`", "", "| metric | value |", "|---|---|"]
    for m in METRICS:
        if m in h:
            i = h.index(m)
            out.append(f"| {m} | {v[i]} {u[i]} |")
    return out


def stall_mix(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = collections.Counter()
    for r in rows[2:]:
        for c in cols:
            try:
                tot[c] += int(r[h.index(c)] or 0)
            except ValueError:
                pass
    s = sum(tot.values()) or 1
    mix = ", ".join(f"{c[6:]} {100 * v / s:.0f}%" for c, v in tot.most_common(7) if v)
    return [f"| stall mix (pc sampling, {s} samples) | {mix} |"]


if __name__ == "__main__":
    raw, sass = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None
    lines = raw_table(raw) + (stall_mix(sass) if sass else [])
    print("\n".join(lines) + "\n")
