"""Executed-instruction and stall-sample profile of a kernel's SASS from an .ncu-rep
(`ncu --page source --print-source sass`), split into regions at labels/branches
(development aid). Usage: ncu_sass_regions.py rep.ncu-rep [min_share]"""
import csv
import subprocess
import sys


def main(rep, min_share=0.01):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    hdr = rows[0]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex = hdr.index("Instructions Executed")
    ism = hdr.index("Warp Stall Sampling (All Samples)")
    recs = []
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        recs.append((r[isrc].strip(), int(r[iex] or 0), int(r[ism] or 0)))
    tot_ex = sum(x[1] for x in recs) or 1
    tot_sm = sum(x[2] for x in recs) or 1
    # region = maximal run of instructions with the same execution count
    i = 0
    n = len(recs)
    print(f"total executed {tot_ex}, samples {tot_sm}, static {n}")
    while i < n:
        j = i
        while j + 1 < n and recs[j + 1][1] == recs[i][1]:
            j += 1
        ex = sum(x[1] for x in recs[i:j + 1])
        sm = sum(x[2] for x in recs[i:j + 1])
        if ex / tot_ex >= min_share or sm / tot_sm >= min_share:
            ops = {}
            for s, _, _ in recs[i:j + 1]:
                t = s.split()
                op = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?")).split(".")[0]
                ops[op] = ops.get(op, 0) + 1
            top = ", ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:8])
            print(f"[{i:5d}-{j:5d}] n={j - i + 1:4d} exec/inst={recs[i][1]:9d} "
                  f"exec%={100 * ex / tot_ex:5.1f} stall%={100 * sm / tot_sm:5.1f}  {top}")
        i = j + 1


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.01)
