"""Summarise an .ncu-rep (ncu --set full) into a JSON file for profiles/: per captured
launch the duration, DRAM bytes (and per cell when --cells is given), issue / pipe
utilisation, registers, occupancy limits and the warp-stall breakdown.
Usage: ncu_to_json.py rep.ncu-rep out.json "source description" [--cells N]"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, out, source, cells=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    res = {"source": source, "kernels": []}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d["Kernel Name"].split("(")[0].replace("dcg::<unnamed>::", "")}
        for key in KEYS:
            if key in d:
                try:
                    k[key] = [float(d[key].replace(",", "")), units[hdr.index(key)]]
                except ValueError:
                    k[key] = [d[key], units[hdr.index(key)]]
        rb = k.get("dram__bytes_read.sum"), k.get("dram__bytes_write.sum")
        if all(isinstance(x, list) and isinstance(x[0], float) for x in rb):
            tot = rb[0][0] * SCALE.get(rb[0][1], 1) + rb[1][0] * SCALE.get(rb[1][1], 1)
            k["dram_bytes"] = tot
            if cells:
                k["dram_bytes_per_cell"] = tot / cells
        st = {}
        for h in hdr:
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(d[h])
                except ValueError:
                    continue
                if v > 0.02:
                    st[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        k["stalls_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1]))
        res["kernels"].append(k)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    cells = None
    if "--cells" in sys.argv:
        i = sys.argv.index("--cells")
        cells = float(sys.argv[i + 1])
        del sys.argv[i:i + 2]
    main(sys.argv[1], sys.argv[2], sys.argv[3], cells)
