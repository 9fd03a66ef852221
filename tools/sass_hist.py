"""Opcode histogram of the hottest loop of a kernel in a cuobjdump -sass listing
(development aid). Usage: sass_hist.py listing.sass name_substring"""
import re
import sys
from collections import Counter


def main():
    text = open(sys.argv[1]).read()
    funcs = re.split(r"\n\s+Function : ", text)
    body = next(f for f in funcs[1:] if sys.argv[2] in f.split("\n", 1)[0])
    ins = []
    for line in body.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    best = None  # largest backward branch = main loop
    for i, (a, s) in enumerate(ins):
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*)?0x([0-9a-f]+)", s) or re.search(r"BRA .*?0x([0-9a-f]+)", s)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and tgt in addr and (best is None or i - addr[tgt] > best[1] - best[0]):
                best = (addr[tgt], i)
    lo, hi = best if best else (0, len(ins) - 1)
    c = Counter()
    for _, s in ins[lo:hi + 1]:
        op = s.split()[0]
        if op.startswith("@"):
            op = s.split()[1]
        c[op.split(".")[0]] += 1
    print(f"loop {lo}..{hi}: {hi - lo + 1} instructions")
    for op, n in c.most_common(40):
        print(f"{n:6d} {op}")


if __name__ == "__main__":
    main()
