"""Render profiles/round2_matrix/*.json as the DESIGN.md section 5 table."""
import glob
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/round2_matrix"
rows = []
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    try:
        x = [json.loads(l) for l in open(f) if l.startswith("{")][-1]
    except Exception:
        continue
    r = x.get("roofline") or {}
    e = x.get("e2e") or {}
    rows.append((os.path.basename(f)[:-5], x["value"] / 1e6, x.get("ms_per_step"), x.get("resets_per_step"),
                 r.get("kernel"), r.get("ms_per_launch"), r.get("frac"), r.get("step_frac"),
                 e.get("value", 0) / 1e6, (e.get("delta") or {}).get("value", 0) / 1e6))
print("| config | M env-steps/s | ms/step | resets/step | dominant kernel: ms, frac of HBM | step frac | e2e dense / delta (M) |")
print("|---|---|---|---|---|---|---|")
for n, v, ms, rps, k, kms, fr, sf, e, dl in rows:
    print(f"| {n} | {v:.2f} | {ms} | {rps} | {k}: {kms}, {fr} | {sf} | {e:.2f} / {dl:.2f} |")
