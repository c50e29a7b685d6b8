"""Instruction mix of the hot loops of one kernel in the built library.

    python tools/sass_loops.py <kernel-name-substring> [--min-bytes 0x300] [--dump LO HI]

Lists every backward branch spanning at least --min-bytes with the opcode
histogram of its body (the loop), to check SASS before spending GPU time.
"""
import argparse
import collections
import re
import subprocess

import os
LIB = os.environ.get("SASS_LIB", "paper_2106_12270_b200/libaliaskit_b200.so")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kernel")
    ap.add_argument("--min-bytes", type=lambda x: int(x, 0), default=0x300)
    ap.add_argument("--dump", nargs=2, type=lambda x: int(x, 16))
    a = ap.parse_args()
    L = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout.split("\n")
    st = [i for i, l in enumerate(L) if "Function :" in l and a.kernel in l]
    if not st:
        raise SystemExit("kernel not found")
    st = st[0]
    en = next((i for i, l in enumerate(L) if "Function :" in l and i > st), len(L))
    F = []
    for l in L[st:en]:
        m = re.search(r"/\*([0-9a-f]{4,5})\*/\s*(.*?);", l)
        if m:
            F.append((int(m.group(1), 16), re.sub(r"\s+", " ", m.group(2)).strip()))
    if a.dump:
        for ad, t in F:
            if a.dump[0] <= ad <= a.dump[1]:
                print(f"{ad:05x} {t}")
        return
    for ad, t in F:
        m = re.search(r"BRA.*?(0x[0-9a-f]+)", t)
        if m:
            tg = int(m.group(1), 16)
            if tg < ad and ad - tg >= a.min_bytes:
                body = [x for y, x in F if tg <= y <= ad]
                ops = collections.Counter((x.split()[1] if x.startswith("@") else x.split()[0]).split(".")[0]
                                          for x in body)
                print(f"{tg:05x}-{ad:05x} {len(body)} instr: {dict(ops)}")


if __name__ == "__main__":
    main()
