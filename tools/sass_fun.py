"""Opcode histogram / listing of one kernel in a cubin or .so (offline SASS inspection).
Usage: python tools/sass_fun.py LIB FUNC_REGEX [--list] [--loops]
--loops prints every backward branch with its body length (instructions between the
target and the branch), a cheap way to size the hot loop without a GPU."""
import re, subprocess, sys, collections

lib, fre = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs, cur, name = {}, [], None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        if name: funcs[name] = cur
        name, cur = m.group(1), []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and name:
        cur.append((int(m.group(1), 16), m.group(2).strip()))
if name: funcs[name] = cur
for fn, ins in funcs.items():
    if not re.search(fre, fn):
        continue
    print(f"== {fn}: {len(ins)} instructions")
    def op(t):
        t = re.sub(r"^@!?U?P\w+\s+", "", t)
        return t.split()[0].split(".")[0]
    if "--loops" in sys.argv:
        addr = {a: i for i, (a, _) in enumerate(ins)}
        for i, (a, t) in enumerate(ins):
            m = re.search(r"BRA\s+(?:`?\(?\.?L?_?x?)?(0x[0-9a-f]+)", t)
            if m:
                tgt = int(m.group(1), 16)
                if tgt < a and tgt in addr:
                    body = ins[addr[tgt]:i + 1]
                    c = collections.Counter(op(x) for _, x in body)
                    print(f"  loop {tgt:#x}..{a:#x}: {len(body)} instr; " + ", ".join(f"{k} {v}" for k, v in c.most_common(12)))
    else:
        c = collections.Counter(op(t) for _, t in ins)
        print("  " + ", ".join(f"{k} {v}" for k, v in c.most_common(40)))
    if "--list" in sys.argv:
        for a, t in ins:
            print(f"  {a:#06x} {t}")
