"""Summarise ncu outputs into profiles/ (launch-list shares; per-kernel SOL + traffic)."""
import collections
import csv
import json
import subprocess
import sys


def kname(full):
    """'void ns::<unnamed>::foo_kernel<(int)1, ns::<unnamed>::PK>(args)' -> 'foo_kernel<1, PK>'."""
    head = full.replace("dcg::<unnamed>::", "").replace("(anonymous namespace)::", "")
    head = head.replace("unnamed>::", "").replace("dcg::", "").replace("(int)", "")
    depth, cut = 0, len(head)
    for i, ch in enumerate(head):  # cut the argument list: first '(' outside template args
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            cut = i
            break
    head = head[:cut].strip()
    if head.startswith("void "):
        head = head[5:]
    return head


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = kname(d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                 "ms": 1e3, "second": 1e6, "s": 1e6}.get(unit, 1.0)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k, "launches": n, "total_us": round(t, 2),
                    "avg_us": round(t / n, 2), "share": round(t / tot, 4)})
    return out, tot


def rep_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__inst_executed.sum", "launch__grid_size"]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for w, i in idx.items():
            v = r[i]
            if w != "Kernel Name":
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                d[w] = [v, units[i]]
            else:
                d[w] = v.split("(")[0]
        res.append(d)
    return res


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        sh, tot = launch_shares(sys.argv[2])
        print(json.dumps({"total_us": round(tot, 1), "kernels": sh}, indent=1))
    else:
        print(json.dumps(rep_metrics(sys.argv[2]), indent=1))
