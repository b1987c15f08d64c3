"""Per-source-line SASS opcode mix of one kernel from an ncu report (source page,
cuda+sass correlation): warp-instructions per 32 voxels by line, split into classes
(int/address, move, fp, memory, control).  usage: ncu_opmix.py REPORT KERNEL VOXELS [N]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kern, vox = sys.argv[1], sys.argv[2], float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
CLS = {"int": {"IMAD", "IADD3", "LOP3", "ISETP", "LEA", "SHF", "SEL", "VIADD", "VIMNMX", "VIADDMNMX", "IMNMX", "LEA.HI",
               "POPC", "FLO", "BREV", "IABS", "PRMT", "ULEA", "UIADD3", "ULOP3", "UISETP", "USEL", "USHF", "UIMAD", "PLOP3"},
       "move": {"MOV", "UMOV", "S2R", "S2UR", "LDC", "LDCU", "CS2R", "R2UR"},
       "fp": {"FFMA", "FFMA2", "FADD", "FADD2", "FMUL", "FMUL2", "FMNMX", "FMNMX3", "FSEL", "FSETP", "I2FP", "F2I", "FRND",
              "HFMA2", "DADD", "DMUL", "DFMA", "F2F", "I2F", "MUFU", "FCHK", "DSETP"},
       "mem": {"LDG", "STG", "LDS", "STS", "ATOMS", "ATOMG", "RED", "REDG", "LDL", "STL", "SHFL", "REDUX", "VOTE", "LDSM",
               "LD", "ST", "MATCH", "ATOM"},
       "ctrl": {"BRA", "BSSY", "BSYNC", "WARPSYNC", "BAR", "EXIT", "NOP", "CALL", "RET", "YIELD", "BMOV", "JMP", "BPT"}}
cls_of = {op: c for c, ops in CLS.items() for op in ops}
lines = collections.defaultdict(lambda: collections.Counter())
src = {}
cur = None
for blk in raw.split('"File Path"')[1:]:
    rows = list(csv.reader(io.StringIO('"File Path"' + blk)))
    fname = rows[0][1].split("/")[-1] if len(rows[0]) > 1 else "?"
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
    if not hi:
        continue
    h = rows[hi[0]]
    ie = h.index("Instructions Executed")
    for r in rows[hi[0] + 1:]:
        if len(r) <= ie:
            continue
        if r[0]:
            cur = (fname, int(r[0]))
            src[cur] = r[1].strip()[:70]
            continue
        if cur is None:
            continue
        s = re.sub(r"^@!?U?P\w+\s+", "", r[3].strip())
        op = s.split()[0].split(".")[0] if s else "?"
        try:
            n = float(r[ie])
        except ValueError:
            continue
        lines[cur][cls_of.get(op, "other")] += n
        lines[cur]["_" + op] += n
g = vox / 32
tot = collections.Counter()
for c in lines.values():
    for k, v in c.items():
        if not k.startswith("_"):
            tot[k] += v
print("per 32 voxels:", {k: round(v / g, 1) for k, v in tot.most_common()}, "total", round(sum(tot.values()) / g, 1))
rank = sorted(lines.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if not k.startswith("_")))
for (f, ln), c in rank[:top]:
    t = sum(v for k, v in c.items() if not k.startswith("_"))
    ops = ", ".join(f"{k[1:]} {v / g:.1f}" for k, v in c.most_common() if k.startswith("_"))[:90]
    print(f"{f[:14]:14s} L{ln:5d} {t / g:6.1f}  {src[(f, ln)][:60]:60s} | {ops}")
