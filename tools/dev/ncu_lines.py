"""Aggregate an ncu source page (cuda,sass) per CUDA source line."""
import csv, sys, collections, subprocess, io, os

def lines(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, *(["--launch-skip", os.environ["NCU_SKIP"], "--launch-count", "1"] if os.environ.get("NCU_SKIP") else []), "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    fpath = ""; cur = None; hdr = None
    for r in rows:
        if not r: continue
        if r[0] == "File Path": fpath = r[1].split("/")[-1]; continue
        if r[0] == "Function Name": continue
        if r[0] == "Line No": hdr = r; si = hdr.index("Warp Stall Sampling (All Samples)"); ii = hdr.index("Instructions Executed"); continue
        if hdr is None: continue
        if r[0]:
            cur = (fpath, r[0]); agg[cur][2] = r[1][:100]
        if cur is None or len(r) <= ii: continue
        try:
            agg[cur][0] += float(r[si] or 0); agg[cur][1] += float(r[ii] or 0)
        except ValueError:
            pass
    ts = sum(v[0] for v in agg.values()) or 1; ti = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"stall {v[0]/ts:6.3f} inst {v[1]/ti:6.3f}  {k[0]}:{k[1]:<5} {v[2]}")

if __name__ == "__main__":
    lines(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
