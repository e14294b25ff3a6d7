"""Summarise an ncu report (read here, no GPU): top SASS opcodes with their
stall samples, the hottest instructions, stall reasons and key throughputs.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source",
                                           "sass"))))
    h = rows[1]
    isrc, iex = h.index("Source"), h.index("Instructions Executed")
    ist = h.index("Warp Stall Sampling (All Samples)")
    by, st, hot, tot, tots = collections.Counter(), collections.Counter(), [], 0, 0
    for r in rows[2:]:
        try:
            n, s = int(r[iex] or 0), int(r[ist] or 0)
        except ValueError:
            continue
        f = r[isrc].split()
        op = (f[1] if f and f[0].startswith("@") else f[0] if f else "").split(".")[0]
        by[op] += n
        st[op] += s
        tot += n
        tots += s
        hot.append((s, n, r[isrc][:72]))
    print(f"instructions {tot}  stall samples {tots}")
    for op, n in by.most_common(16):
        print(f"  {op:10s} {n:13d} {n / tot * 100:5.1f}%  stall {st[op] / max(tots, 1) * 100:5.1f}%")
    print("hottest:")
    for x in sorted(hot, reverse=True)[:10]:
        print("  ", x)
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    names, vals = raw[0], raw[2]
    keep = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
            "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
            "lts__t_bytes.sum", "smsp__inst_executed.sum",
            # L2 -> SM traffic (the TMA window staging) and L2 sector load
            "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
            "lts__t_sectors.sum.pct_of_peak_sustained_elapsed")
    print("metrics:")
    for i, n in enumerate(names):
        if n in keep:
            print(f"  {n} = {vals[i]} {raw[1][i]}")
    print("stall reasons (samples):")
    sr = []
    for i, n in enumerate(names):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                sr.append((float(vals[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    for v, n in sorted(sr, reverse=True)[:10]:
        print(f"  {n:28s} {v:10.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
