"""Instruction mix of a kernel's hottest straight-line region, from cuobjdump -sass.

    cuobjdump -sass -fun <mangled> lib.so > k.sass   (or a whole-cubin dump + --kernel)
    python scripts/sass_mix.py k.sass [--kernel SUBSTR] [--per-term-sts N] [--excerpt OUT]

The region is the branch-free run (between BRA/EXIT/labels) with the most
shared stores; terms = STS count / per-term-sts (2 for the 96-bit slot RMW:
STS + STS.64).  Pipes: ALU = integer logic/shift/add/min-max, FMA = IMAD/FP32,
LSU = LDS/STS/LDG.  --excerpt writes the region itself (for profiles/).
"""
from __future__ import annotations

import argparse
import re
from collections import Counter

ALU = {"IADD3", "LOP3", "SHF", "SEL", "ISETP", "LEA", "VIMNMX", "VIMNMX3", "IMNMX", "PRMT", "FLO",
       "POPC", "PLOP3", "P2R", "R2P", "IADD", "VOTE", "MOV", "UMOV"}
FMA = {"IMAD", "FFMA", "FMUL", "FADD"}
LSU = {"LDS", "STS", "LDG", "STG", "LD", "ST", "UBLKPF", "ATOMS", "REDG"}


def instructions(path: str, kernel: str | None):
    cur, keep = [], kernel is None
    for raw in open(path):
        if "Function :" in raw:
            keep = kernel is None or kernel in raw
            continue
        if not keep:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", raw)
        if not m:
            continue
        text = m.group(1).strip()
        if text.startswith("NOP"):
            continue
        cur.append(text)
    return cur


def opcode(text: str) -> str:
    return re.sub(r"^@!?U?P[T0-9]+\s+", "", text).split()[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sass")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--per-term-sts", type=float, default=2.0)
    ap.add_argument("--excerpt", default=None)
    a = ap.parse_args()
    ins = instructions(a.sass, a.kernel)
    best, cur = [], []
    for t in ins:
        op = opcode(t)
        cur.append(t)
        if op.startswith(("BRA", "EXIT", "RET", "BSYNC", "WARPSYNC")):
            if sum(opcode(x).startswith("STS") for x in cur) > sum(opcode(x).startswith("STS") for x in best):
                best = cur
            cur = []
    ops = Counter(opcode(t) for t in best)
    nsts = sum(v for k, v in ops.items() if k.startswith("STS"))
    terms = nsts / a.per_term_sts if nsts else 1
    print(f"region: {len(best)} instructions, {nsts} STS -> {terms:.0f} terms, "
          f"{len(best) / terms:.2f} instructions/term")
    cls = Counter()
    for k, v in ops.items():
        base = k.split(".")[0]
        cls["alu" if base in ALU else "fma" if base in FMA else "lsu" if base in LSU else base] += v
    print("per term by pipe:", {k: round(v / terms, 2) for k, v in sorted(cls.items())})
    print("per term by opcode:", [(k, round(v / terms, 2)) for k, v in ops.most_common(30)])
    if a.excerpt:
        with open(a.excerpt, "w") as f:
            f.write("\n".join(best) + "\n")


if __name__ == "__main__":
    main()
