"""Per-region and per-helper-line warp-instruction / stall-sample shares of one kernel.
usage: ncu_lines.py REPORT KERNEL VOXELS a:b:name ... [--helpers N]"""
import csv, io, subprocess, sys
rep, kern, vox = sys.argv[1], sys.argv[2], float(sys.argv[3])
args = [x for x in sys.argv[4:] if not x.startswith("--")]
regions = [(int(a), int(b), n) for a, b, n in (r.split(":") for r in args)]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
agg, src = {}, {}
for b in raw.split('"Function Name"')[1:]:
    rows = list(csv.reader(io.StringIO('"Function Name"' + b)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
    if not hi:
        continue
    h = rows[hi[0]]
    ii = h.index("Instructions Executed")
    si = [i for i, x in enumerate(h) if x.startswith("Warp Stall Sampling (All")][0]
    for r in rows[hi[0] + 1:]:
        try:
            ln, v, st = int(r[0]), float(r[ii]), float(r[si])
        except (ValueError, IndexError):
            continue
        a = agg.setdefault(ln, [0, 0]); a[0] += v; a[1] += st; src[ln] = r[1].strip()[:80]
ti = sum(a[0] for a in agg.values()); ts = sum(a[1] for a in agg.values())
print(f"total {ti / (vox / 32):.0f} warp-inst per 32 voxels")
res = {}
for ln, (v, st) in agg.items():
    n = next((n for a, b, n in regions if a <= ln <= b), "helpers")
    r = res.setdefault(n, [0, 0]); r[0] += v; r[1] += st
for n, (v, st) in sorted(res.items(), key=lambda kv: -kv[1][0]):
    print(f"{n:24s} {v / (vox / 32):6.1f} /32vox ({100 * v / ti:4.1f}%)  stalls {100 * st / ts:5.1f}%")
print("-- helper lines")
lo = min(a for a, _, _ in regions)
for ln, (v, st) in sorted(((l, a) for l, a in agg.items() if l < lo), key=lambda kv: -kv[1][0])[:12]:
    print(f"L{ln:5d} {v / (vox / 32):6.1f} /32vox stalls {100 * st / ts:5.1f}%  {src[ln]}")
