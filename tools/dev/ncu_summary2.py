"""Summarise an ncu report (one launch) into a text file for profiles/.

    python tools/dev/ncu_summary2.py <report.ncu-rep> <launch id> <out.txt> [title]

Key Speed-of-Light / memory / scheduler / occupancy metrics, the warp-stall
reasons (sampled), and the source lines with the most executed instructions
and stall samples (needs -lineinfo and --import-source on).
"""
import csv
import io
import subprocess
import sys


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main(rep, lid, out, title=""):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv"))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    det = [r for r in rows[1:] if r[ix["ID"]] == str(lid)]
    lines = [f"# {title or rep}", f"# ncu report {rep}, launch {lid}: {det[0][ix['Kernel Name']]}",
             f"# grid {det[0][ix['Grid Size']]} block {det[0][ix['Block Size']]}", ""]
    keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L1/TEX Cache Throughput",
            "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions",
            "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Achieved Occupancy",
            "Theoretical Occupancy", "Avg. Active Threads Per Warp", "Branch Efficiency", "L2 Hit Rate",
            "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block", "Waves Per SM")
    for r in det:
        if r[ix["Metric Name"]] in keep:
            lines.append(f"{r[ix['Section Name']][:30]:30s} {r[ix['Metric Name']]:38s} {r[ix['Metric Value']]:>14s} {r[ix['Metric Unit']]}")
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    h, units = raw[0], raw[1]
    vals = raw[2 + int(lid)] if len(raw) > 2 + int(lid) else raw[-1]
    lines += ["", "# DRAM bytes (per launch)"]
    for k, u, v in zip(h, units, vals):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            lines.append(f"{k:40s} {v} {u}")
    stalls = []
    for k, v in zip(h, vals):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                stalls.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    lines += ["", "# warp stall samples (share)"]
    for s, k in sorted(stalls, reverse=True)[:12]:
        lines.append(f"{k:32s} {100 * s / tot:6.1f} %")
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                                          "--launch-skip", str(lid), "--launch-count", "1"))))
    res, hdr2, fname = [], None, ""
    for r in src:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr2 = r
            continue
        if hdr2 is None or len(r) < 8 or not r[0]:
            continue
        try:
            res.append((f"{fname}:{r[0]}", int(r[7] or 0), int(r[4] or 0), r[1].strip()[:100]))
        except ValueError:
            pass
    ti = sum(x[1] for x in res) or 1
    ts = sum(x[2] for x in res) or 1
    lines += ["", "# source lines by executed (warp) instructions: line, instr %, stall-sample %, source"]
    for ln, ins, st, s in sorted(res, key=lambda x: -x[1])[:20]:
        lines.append(f"{ln:>18s} {100 * ins / ti:5.1f} {100 * st / ts:5.1f}  {s}")
    lines += ["", "# source lines by stall samples"]
    for ln, ins, st, s in sorted(res, key=lambda x: -x[2])[:15]:
        lines.append(f"{ln:>18s} {100 * ins / ti:5.1f} {100 * st / ts:5.1f}  {s}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
