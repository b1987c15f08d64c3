"""Per-source-line warp-instruction counts of one kernel in an ncu report."""
import csv, subprocess, io, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
vox = float(sys.argv[4]) if len(sys.argv) > 4 else 512 * 512 * 320
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
agg = {}
for b in raw.split('"Function Name"')[1:]:
    rows = list(csv.reader(io.StringIO('"Function Name"' + b)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
    if not hi:
        continue
    hdr = rows[hi[0]]
    ii = hdr.index("Instructions Executed")
    for r in rows[hi[0] + 1:]:
        if len(r) > ii and r[0]:
            try:
                v = float(r[ii])
            except ValueError:
                continue
            k = (r[0], r[1].strip()[:100])
            agg[k] = agg.get(k, 0) + v
tot = sum(agg.values())
print(f"total {tot:.3e}  per 32 voxels {tot / (vox / 32):.0f}")
for (ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"L{ln:>5} {v / tot * 100:5.1f}% {v / (vox / 32):6.1f}  {src}")
