"""Aggregate an ncu source page per enclosing function of gr_step.cu (dev helper).

    python tools/dev/ncu_funcs.py report.ncu-rep [source.cu]
"""
import collections, csv, io, re, subprocess, sys


def main(rep, src_path="paper_2402_16801_b200/csrc/gr_step.cu", top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    src = open(src_path).read().splitlines()
    base = src_path.split("/")[-1]
    starts = []
    for n, line in enumerate(src, 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?(\w+)\s*\(", line)
        if m:
            starts.append((n, m.group(1)))

    def fn(line):
        best = "?"
        for n, name in starts:
            if n <= line:
                best = name
        return best

    agg = collections.defaultdict(lambda: [0.0, 0.0])
    fpath, hdr, cur = "", None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fpath = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            si = hdr.index("Warp Stall Sampling (All Samples)")
            ii = hdr.index("Instructions Executed")
            continue
        if hdr is None:
            continue
        if r[0]:
            try:
                cur = (fpath, int(r[0]))
            except ValueError:
                cur = None
        if cur is None or len(r) <= ii:
            continue
        try:
            key = fn(cur[1]) if cur[0] == base else cur[0]
            agg[key][0] += float(r[si] or 0)
            agg[key][1] += float(r[ii] or 0)
        except ValueError:
            pass
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print("stall  inst   function")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{v[0] / ts:6.3f} {v[1] / ti:6.3f}  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])
