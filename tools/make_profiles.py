"""Summarise one GPU round's ncu outputs (tools/gpu_round.sh) into profiles/ (tracked).

Usage: python tools/make_profiles.py TAG   (reads gpurun_out/launches_TAG.csv and
gpurun_out/full_*_TAG.ncu-rep)"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import launch_shares  # noqa: E402

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_inst_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__occupancy_limit_registers": "ctas_per_sm_by_regs",
    "sm__cycles_active.avg": "sm_active_cycles",
    "gpc__cycles_elapsed.max": "elapsed_cycles",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3}


def rep_rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d["Kernel Name"].split("(")[0].replace("dcg::<unnamed>::", "")}
        for k, name in KEYS.items():
            if k not in d:
                continue
            u = units[hdr.index(k)]
            try:
                v = float(d[k].replace(",", ""))
            except ValueError:
                continue
            if name.startswith("dram_read") or name.startswith("dram_write"):
                v *= SCALE.get(u, 1)
            elif name == "duration":
                v *= SCALE.get(u, 1)  # -> us
            rec[name] = round(v, 3)
        st = {}
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio"):
                try:
                    v = float(d[k])
                except ValueError:
                    continue
                if v >= 0.05:
                    st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        if rec.get("sm_active_cycles") and rec.get("elapsed_cycles"):
            # share of the launch the SMs had resident CTAs (ramp + drain = the rest)
            rec["sm_active_frac"] = round(rec["sm_active_cycles"] / rec["elapsed_cycles"], 4)
        rec["stalls_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1]))
        out.append(rec)
    return out


def main(tag):
    g = os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    sh, tot = launch_shares(os.path.join(g, f"launches_{tag}.csv"))
    json.dump({"source": f"ncu --metrics gpu__time_duration.sum --clock-control none, DC_NO_GRAPH=1 "
                         f"tools/profile_cycle.py --cycles 2 (100 members, 500x300, 64 drifters); "
                         f"serialised cold-cache launches", "total_us": round(tot, 1),
               "kernels": sh}, open(os.path.join(prof, "r1_launches_cycle.json"), "w"), indent=1)
    import shutil
    shutil.copy(os.path.join(g, f"launches_{tag}.csv"), os.path.join(prof, "r1_launches_cycle.csv"))
    groups = {"swe": "r1_swe_stage_ncu.json", "q_half_apply": "r1_perturb_ncu.json",
              "pull_apply": "r1_analysis_ncu.json", "local_blocks": "r1_local_blocks_ncu.json",
              "philox_soar": "r1_philox_soar_ncu.json", "cfl_scan": "r1_cfl_scan_ncu.json"}
    for key, fn in groups.items():
        rep = os.path.join(g, f"full_{key}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            continue
        rows = rep_rows(rep)
        json.dump({"source": f"ncu --set full --clock-control none ({os.path.basename(rep)})",
                   "launches": rows}, open(os.path.join(prof, fn), "w"), indent=1)
        if key == "swe":
            n = len(rows)
            traffic = sum(r["dram_read"] + r["dram_write"] for r in rows) / n
            json.dump({"dram_bytes_per_launch": traffic,
                       "per_stage": {r["kernel"]: r["dram_read"] + r["dram_write"] for r in rows},
                       "source": os.path.basename(rep),
                       "note": "mean over the captured stage-1 and stage-2 launches"},
                      open(os.path.join(prof, "swe_stage_traffic.json"), "w"), indent=1)
    print("wrote profiles for", tag)


if __name__ == "__main__":
    main(sys.argv[1])
