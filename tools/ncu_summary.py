"""Key counters and the warp-stall breakdown of every kernel in an ncu report (ncu --set full).
    python tools/ncu_summary.py REPORT.ncu-rep [markdown]"""
import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__shared_mem_per_block",
        "launch__grid_size", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum"]


def summary(rep, md=False):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        lines.append(f"### {r[h.index('Kernel Name')]}" if md else r[h.index('Kernel Name')])
        if md:
            lines += ["", "| metric | value |", "|---|---|"]
        for k in KEYS:
            if k in h:
                v = f"{r[h.index(k)]} {u[h.index(k)]}".strip()
                lines.append(f"| `{k}` | {v} |" if md else f"  {k:80s} {v}")
        st = [(k, float(r[i].replace(",", "") or 0)) for i, k in enumerate(h)
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1.0
        top = sorted(st, key=lambda kv: -kv[1])[:8]
        s = ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.1f}%" for k, v in top)
        lines.append(("" if not md else "\nWarp stall samples: ") + s if md else "  stalls: " + s)
        lines.append("")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summary(sys.argv[1], len(sys.argv) > 2))
