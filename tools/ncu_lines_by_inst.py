"""Per-source-line executed instructions of one kernel in an ncu report (sorted by count),
plus sums over line ranges.  Usage: python tools/ncu_lines_by_inst.py REP KERNEL_REGEX FILE [N]"""
import csv, io, subprocess, sys

rep, kre, fname = sys.argv[1], sys.argv[2], sys.argv[3]
ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
for b in raw.split('"File Path"')[1:]:
    rows = list(csv.reader(io.StringIO('"File Path"' + b)))
    if fname not in rows[0][1]:
        continue
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
    hdr = rows[hi]
    ii = hdr.index("Instructions Executed")
    wi = hdr.index("Warp Stall Sampling (All Samples)")
    def f(x):
        try:
            return float(x)
        except Exception:
            return 0.0
    lines = [r for r in rows[hi + 1:] if r and r[0].isdigit()]
    tot = sum(f(r[ii]) for r in lines)
    stot = sum(f(r[wi]) for r in lines) or 1
    print(f"total {tot:.4e}")
    for r in sorted(lines, key=lambda r: -f(r[ii]))[:ntop]:
        print(f"L{r[0]:>4} inst {f(r[ii]) / tot * 100:5.2f}% stall {f(r[wi]) / stot * 100:5.2f}%  {r[1].strip()[:100]}")
