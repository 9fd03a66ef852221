"""Stall samples per SASS opcode of one kernel in an .ncu-rep (development aid):
which instruction classes the warps are stuck on, by reason.
Usage: ncu_opcode_stalls.py source.csv [kernel_index]   (source.csv from
`ncu -i rep --page source --csv --print-source sass`)"""
import collections
import csv
import sys

REASONS = ["stall_wait", "stall_math", "stall_dispatch", "stall_barrier", "stall_not_selected",
           "stall_selected", "stall_long_sb", "stall_short_sb", "stall_no_inst", "stall_branch_resolving"]


def main(path, which=0):
    blocks, cur = [], None
    for ln in open(path).read().splitlines():
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            blocks.append(cur)
        elif cur is not None:
            cur.append(ln)
    b = blocks[which]
    print(b[0][:100])
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    idx = {r: hdr.index(r) for r in REASONS}
    acc = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        s = r[isrc].strip().split()
        if not s:
            continue
        op = s[1] if s[0].startswith("@") and len(s) > 1 else s[0]
        op = op.split(".")[0]
        acc[op]["exec"] += int(r[iex] or 0)
        for k, i in idx.items():
            v = int(r[i] or 0)
            acc[op][k] += v
            tot[k] += v
    allsum = sum(tot.values()) or 1
    print("total samples", allsum, {k[6:]: round(v / allsum, 3) for k, v in tot.most_common()})
    ex_tot = sum(a["exec"] for a in acc.values()) or 1
    for op, a in sorted(acc.items(), key=lambda x: -sum(v for k, v in x[1].items() if k != "exec"))[:18]:
        s = sum(v for k, v in a.items() if k != "exec")
        top = ", ".join(f"{k[6:]} {v / allsum:.3f}" for k, v in a.most_common() if k != "exec" and v)
        print(f"{op:10s} exec {a['exec'] / ex_tot:.3f} samples {s / allsum:.3f}: {top[:150]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
