"""Per-row opcode histogram of a streaming stage kernel in a cuobjdump -sass listing
(development aid): rows are delimited by every third BAR.SYNC (3 barriers per row).
Usage: sass_rows.py listing.sass name_substring [name_substring ...]"""
import re
import sys
from collections import Counter


def rows(text, name):
    funcs = re.split(r"\n\s+Function : ", text)
    body = next(f for f in funcs[1:] if name in f.split("\n", 1)[0])
    ins = []
    for line in body.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append(m.group(2).strip())
    bars = [i for i, s in enumerate(ins) if "BAR.SYNC" in s]
    out = []
    for r in range(1, len(bars) // 3):
        lo, hi = bars[3 * r - 1] + 1, bars[3 * r + 2]
        c = Counter()
        for s in ins[lo:hi + 1]:
            op = s.split()[0]
            if op.startswith("@"):
                op = s.split()[1]
            c[op.split(".")[0]] += 1
        out.append(c)
    return out


def main():
    text = open(sys.argv[1]).read()
    for name in sys.argv[2:]:
        rs = rows(text, name)
        tots = [sum(c.values()) for c in rs]
        print(name, "rows", len(rs), "instr/row", tots)
        if rs:
            c = rs[len(rs) // 2]
            print("   ", ", ".join(f"{op}:{n}" for op, n in c.most_common(34)))


if __name__ == "__main__":
    main()
