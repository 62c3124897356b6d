#!/usr/bin/env python
"""SASS evidence for the hot kernels of libasse.so (cuobjdump, no GPU needed): per kernel
the mnemonic histogram of the instructions that prove the Blackwell-native data movement
(UBLKCP = cp.async.bulk / TMA bulk copies, SYNCS = mbarrier ops, ATOMS = shared-memory
atomics, REDUX = warp reductions, PRMT = byte permutes) and an excerpt of the hot loops.

  python tools/sass_excerpt.py > profiles/r02_sass_hot_loops.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1807_01527_b200", "libasse.so")
KERNELS = [
    ("k_scan_own (C3-C5 geometry, u8)", r"k_scan_own.*GeoCt.*Li1ELb0E|k_scan_ownILi1ELb0ENS_5GeoCt"),
    ("k_fold<1,5> (u8, g = 512)", r"k_foldILi1ELi5ELb0ELi0E"),
    ("k_fold<2,5> (u16, g = 512)", r"k_foldILi2ELi5ELb0ELi0E"),
]
MNEM = ["UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "ATOMS", "ATOMG", "RED", "REDUX", "PRMT", "LDS", "STS",
        "LDG", "STG", "BAR", "NANOSLEEP", "CCTL", "MEMBAR"]


def functions():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs, cur, name = {}, [], None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = cur
            name, cur = m.group(1), []
        elif name and instr(line):
            cur.append(line)
    if name:
        funcs[name] = cur
    return funcs


def instr(line):
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    return m.group(2) if m else None


def main():
    funcs = functions()
    for title, pat in KERNELS:
        names = [n for n in funcs if re.search(pat, n)]
        if not names:
            print("## %s: not found\n" % title)
            continue
        name = names[0]
        body = funcs[name]
        hist = collections.Counter()
        for line in body:
            op = instr(line)
            if op:
                base = op.split(".")[0]
                for mn in MNEM:
                    if base == mn:
                        hist[op] += 1
        print("## %s\n\nfunction %s, %d SASS lines\n" % (title, name, len(body)))
        for k, v in sorted(hist.items()):
            print("  %-40s %d" % (k, v))
        # hot-loop excerpt: the densest window of ATOMS / UBLKCP / PRMT / REDUX instructions
        marks = [i for i, l in enumerate(body) if (instr(l) or "").split(".")[0] in ("ATOMS", "UBLKCP", "PRMT", "REDUX")]
        if marks:
            best, bi = 0, marks[0]
            for i in marks:
                c = sum(1 for j in marks if i <= j < i + 80)
                if c > best:
                    best, bi = c, i
            print("\nexcerpt (densest 80-line window, %d marked instructions):\n" % best)
            for l in body[max(0, bi - 10):bi + 80]:
                print("  " + re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", l).strip())
        print()


if __name__ == "__main__":
    sys.exit(main())
