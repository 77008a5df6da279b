"""Dynamic SASS opcode mix of the profiled kernel, per (gate x CMux), and the source lines that execute
the most non-FP64 instructions.   python tools/ncu_mix.py rep.ncu-rep GATES [N]"""
import csv, io, subprocess, sys
from collections import Counter, defaultdict
rep, gates = sys.argv[1], int(sys.argv[2]); N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
per = gates * 500
def export(src):
    t = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", src], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(t)))
rows = export("sass")
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]; col = {h: i for i, h in enumerate(hdr)}
ex = {}
def opcode(src):
    p = src.split()
    return (p[1] if src.startswith("@") else p[0]).rstrip(";")
mix = Counter()
for r in rows[hi + 1:]:
    if len(r) == len(hdr):
        n = float(r[col["Instructions Executed"]]); s = r[col["Source"]].strip()
        ex[r[0]] = (n, s); mix[opcode(s)] += n
tot = sum(mix.values())
fp64 = sum(n for o, n in mix.items() if o.split(".")[0] in ("DADD", "DMUL", "DFMA"))
print(f"total {tot/per:.0f} instr per gate-CMux, FP64 {fp64/per:.0f}, other {(tot-fp64)/per:.0f}")
print(" ".join(f"{o}={n/per:.0f}" for o, n in mix.most_common(32)))
rows = export("cuda,sass")
cur = None; fname = None; by = defaultdict(float)
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if len(r) >= 4 and r[0].strip().isdigit(): cur = (fname, int(r[0]), r[1].strip()[:80]); continue
    if len(r) >= 4 and r[2].startswith("0x") and cur:
        n, s = ex.get(r[2], (0, ""))
        if s and opcode(s).split(".")[0] not in ("DADD", "DMUL", "DFMA"): by[cur] += n
for k, n in sorted(by.items(), key=lambda kv: -kv[1])[:N]:
    print(f"{n/per:7.1f}  {k[0]}:{k[1]}  {k[2]}")
