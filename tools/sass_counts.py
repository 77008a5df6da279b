"""Per-kernel counts of the SASS mnemonics that prove which hardware paths libtfhe_b200.so uses.
    python tools/sass_counts.py [--out profiles/r02_sass_counts.txt]
UBLKCP = cp.async.bulk (TMA) copies, SYNCS = mbarrier operations, LDTM / STTM = tensor-memory loads / stores
(tcgen05.ld / st), UTCIMMA / UTCHMMA... = tcgen05.mma, UTCBAR = tcgen05.commit, DFMA / DADD / DMUL = FP64 pipe,
IMAD / IMMA = integer pipe / legacy tensor path, BAR = named barriers, UCGABAR_* = cluster barriers,
STAS = st.async into a peer CTA's shared memory (DSMEM)."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2005_01945_b200", "csrc", "libtfhe_b200.so")
WATCH = ("UBLKCP", "SYNCS", "LDTM", "STTM", "UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "UTCCP", "UTCATOMSWS", "DFMA", "DADD", "DMUL",
         "IMAD", "IMMA", "BAR", "UCGABAR_ARV", "UCGABAR_WAIT", "STAS", "SHFL", "LDS", "STS", "LDG", "STG", "ATOMS", "REDUX")


def main():
    text = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kernels, name = collections.OrderedDict(), None
    for line in text.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip().split("(")[0]
            kernels[name] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and name:
            kernels[name][m.group(1)] += 1
    lines = [f"# cuobjdump -sass counts per kernel of {os.path.relpath(LIB, ROOT)} (static instruction counts)"]
    for kname, cnt in kernels.items():
        shown = ", ".join(f"{op} {cnt[op]}" for op in WATCH if cnt[op])
        lines.append(f"{kname}: total {sum(cnt.values())}; {shown}")
    body = "\n".join(lines)
    print(body)
    if "--out" in sys.argv:
        with open(sys.argv[sys.argv.index("--out") + 1], "w") as f:
            f.write(body + "\n")


if __name__ == "__main__":
    main()
