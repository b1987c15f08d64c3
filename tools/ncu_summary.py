"""Summarise an ncu --set full report: headline metrics per kernel, stall reasons and
the hottest source lines (needs -lineinfo and --import-source on)."""
import csv, subprocess, sys, io

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else "k_pass"
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 20
vox = float(sys.argv[4]) if len(sys.argv) > 4 else 512 * 512 * 320


def run(args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
h = det[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
want = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp"]
seen = {}
for r in det[1:]:
    if kfilter in r[ki] and r[mi] in want:
        seen.setdefault(r[ki], {})[r[mi]] = f"{r[vi]} {r[ui]}"
for k, d in seen.items():
    print(f"== {k}")
    for m in want:
        if m in d:
            print(f"   {m:36s} {d[m]}")
raw = run(["--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kfilter}"])
# the source page prints one block per (kernel, source file): each starts with a
# "File Path" row (the kernel file, or a CUDA header holding an inlined intrinsic)
blocks = raw.split('"File Path"')
for b in blocks[1:]:
    rows = list(csv.reader(io.StringIO('"File Path"' + b)))
    path = rows[0][1].rsplit("/", 1)[-1] if len(rows[0]) > 1 else "?"
    name = (rows[1][1] if len(rows) > 1 and len(rows[1]) > 1 else "?")
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
    if not hi:
        continue
    hdr = rows[hi[0]]
    ii = hdr.index("Instructions Executed")
    wi = hdr.index("Warp Stall Sampling (All Samples)")
    cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
    lines = [r for r in rows[hi[0] + 1:] if len(r) > max(cols) and r[0] not in ("",)]

    def f(x):
        try:
            return float(x)
        except Exception:
            return 0.0
    tot = sum(f(r[ii]) for r in lines)
    stot = sum(f(r[wi]) for r in lines) or 1
    print(f"== {name[:60]} [{path}]: warp-instructions {tot:.3e} = {tot / (vox / 32):.0f} per 32 voxels")
    st = {hdr[i]: sum(f(r[i]) for r in lines) for i in cols}
    print("   stalls: " + ", ".join(f"{k[6:]} {v / stot * 100:.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:7]))
    for r in sorted(lines, key=lambda r: -f(r[wi]))[:ntop]:
        print(f"   L{r[0]:>4} inst {f(r[ii]) / tot * 100:5.1f}% stall {f(r[wi]) / stot * 100:5.1f}%  {r[1].strip()[:90]}")
