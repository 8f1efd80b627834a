"""Summarise an ncu report: duration, DRAM traffic, throughput, occupancy, top stalls."""
import csv, subprocess, sys, io

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__branch_targets_threads_divergent.sum", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
        "sm__warps_active.avg.per_cycle_active"]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        item = {"kernel": d.get("Kernel Name", "")[:60]}
        for k in KEYS:
            if k in d:
                item[k] = f"{d[k]} {u[k]}".strip()
        try:   # SIMT efficiency: active threads per executed warp instruction
            ti = float(d.get("sass__thread_inst_executed_per_opcode_category", "nan").replace(",", ""))
            wi = float(d.get("smsp__inst_executed.sum", "nan").replace(",", ""))
            item["threads_per_warp_instruction"] = f"{ti / wi:.1f} of 32 ({100 * ti / wi / 32:.0f} % SIMT efficiency)"
        except (ValueError, ZeroDivisionError):
            pass
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[h] or 0) for h in hdr
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        tot = sum(stalls.values()) or 1
        item["top_stalls"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:5]}
        res.append(item)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for it in summary(p):
            print(p)
            for k, v in it.items():
                print("   ", k, v)
