"""Warp-instruction counts of one kernel grouped by source-line ranges of srwcr_kernels.cuh.
usage: ncu_regions.py report kernel voxels start:end:name ..."""
import csv, io, subprocess, sys
rep, kern, vox = sys.argv[1], sys.argv[2], float(sys.argv[3])
regions = [(int(a), int(b), n) for a, b, n in (r.split(":") for r in sys.argv[4:])]
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
        try:
            ln, v = int(r[0]), float(r[ii])
        except (ValueError, IndexError):
            continue
        agg[ln] = agg.get(ln, 0) + v
tot = sum(agg.values())
print(f"total per 32 voxels {tot / (vox / 32):.0f}")
acc = {}
for ln, v in agg.items():
    name = next((n for a, b, n in regions if a <= ln <= b), "other(helpers)")
    acc[name] = acc.get(name, 0) + v
for n, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"{n:28s} {v / (vox / 32):7.1f}  {100 * v / tot:5.1f}%")
