"""Top source lines of an ncu report by stall samples and shared-memory conflicts.
    python tools/ncu_hot_lines.py rep.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(text)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
col = {h: i for i, h in enumerate(hdr)}
src = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0].strip().isdigit()]
def num(r, name):
    try: return float(r[col[name]])
    except Exception: return 0.0
tot = sum(num(r, "# Samples") for r in src)
print(f"total samples {tot:.0f}")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in sorted(src, key=lambda r: -num(r, "# Samples"))[:N]:
    st = sorted(((num(r, h), h[6:]) for h in stall_cols), reverse=True)[:3]
    print(f"{num(r,'# Samples')/tot*100:5.1f}%  L{r[0]:>4} inst={num(r,'Instructions Executed'):.3g} confl={num(r,'L1 Conflicts Shared N-Way'):.3g} "
          f"exc_wf={num(r,'L1 Wavefronts Shared Excessive'):.3g} wf={num(r,'L1 Wavefronts Shared'):.3g} "
          + " ".join(f"{n}:{v:.0f}" for v, n in st) + "  | " + r[1].strip()[:90])
