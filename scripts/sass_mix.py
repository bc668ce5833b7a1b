"""Instruction mix of the hottest straight-line region of a SASS dump (between STS)."""
import re
import sys
from collections import Counter

lines = [l.strip() for l in open(sys.argv[1]) if l.strip() and not l.strip().startswith("NOP")]
# find the longest run between two BRA with many STS: use the region with max STS density
best, cur, region = None, [], []
for l in lines:
    cur.append(l)
    if l.startswith("BRA") or "BRA " in l:
        if best is None or sum("STS" in x for x in cur) > sum("STS" in x for x in best):
            best = cur
        cur = []
ops = Counter(re.sub(r"^@!?U?P\d+\s+", "", l).split()[0] for l in best)
nsts = sum(v for k, v in ops.items() if k.startswith("STS"))
terms = nsts / float(sys.argv[2]) if len(sys.argv) > 2 else nsts
print(f"region: {len(best)} instrs, {nsts} STS -> {terms:.0f} terms, {len(best)/terms:.1f} instr/term")
ALU = ("IADD3", "LOP3", "SHF", "SEL", "ISETP", "LEA", "VIMNMX", "IMNMX", "PRMT", "FLO", "POPC", "PLOP3", "P2R", "R2P")
FMA = ("IMAD", "FFMA", "FMUL", "FADD")
cls = Counter()
for k, v in ops.items():
    base = k.split(".")[0]
    c = "alu" if base in ALU else "fma" if base in FMA else "lsu" if base in ("LDS", "STS", "LDG", "STG") else base
    cls[c] += v
print({k: round(v / terms, 2) for k, v in cls.items()})
print(sorted(((round(v / terms, 2), k) for k, v in ops.items()), reverse=True)[:25])
