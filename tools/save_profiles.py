"""Copy the evidence of one tools/gpu_full.sh run from gpurun_out/ into profiles/ (tracked).

    python tools/save_profiles.py r01

- bench JSON lines            -> profiles/<tag>_bench_<name>.json
- ncu launch list (csv + per-kernel summary) -> profiles/<tag>_tf32_launches.csv / _summary.txt
- ncu --set full of the contraction: selected raw metrics -> profiles/<tag>_ncu_contract_tf32.txt,
  and the per-launch DRAM traffic (read + write, averaged over the captured passes) ->
  profiles/traffic_latest.json["C5:3xtf32"], which bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
           "lts__t_sector_hit_rate.pct", "lts__t_sector_op_read_hit_rate.pct"]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    for name in ("default", "f64", "c2", "c3", "c4", "ref", "rstr_u", "rstr_l", "rstr_k"):
        p = os.path.join(OUT, f"bench_{name}.log")
        if not os.path.exists(p):
            continue
        lines = [x for x in open(p) if x.startswith("{")]
        if lines:
            dst = os.path.join(PROF, f"{tag}_bench_{'tf32' if name == 'default' else name}.json")
            open(dst, "w").write(lines[-1])
            print("wrote", dst)
    lc = os.path.join(OUT, "launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(PROF, f"{tag}_tf32_launches.csv"))
        s = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), lc],
                           capture_output=True, text=True).stdout
        open(os.path.join(PROF, f"{tag}_tf32_launches_summary.txt"), "w").write(s)
        print("wrote launch summary")
    rep = os.path.join(OUT, "prof_tf32_final.ncu-rep")
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        lines, traffic = [], []
        for r in rows[2:]:
            kn = r[hdr.index("Kernel Name")]
            lines.append(kn)
            for m in METRICS:
                if m in hdr:
                    i = hdr.index(m)
                    lines.append(f"  {m} = {r[i]} {units[i]}")
            rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
            wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
            traffic.append(rd + wr)
            lines.append(f"  dram read+write per launch = {rd + wr:.0f} B")
        open(os.path.join(PROF, f"{tag}_ncu_contract_tf32.txt"), "w").write("\n".join(lines) + "\n")
        tp = os.path.join(PROF, "traffic_latest.json")
        cur = json.load(open(tp)) if os.path.exists(tp) else {}
        if traffic:
            cur["C5:3xtf32"] = round(sum(traffic) / len(traffic))
            json.dump(cur, open(tp, "w"), indent=1)
            print("traffic", cur)
    # rSTR-K: the N mixing passes of one C4 step (--set full) -> per-step DRAM traffic
    rep = os.path.join(OUT, "prof_ksrft_mix.ncu-rep")
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        lines, tot = [], 0.0
        for r in rows[2:]:
            lines.append(r[hdr.index("Kernel Name")])
            for m in METRICS + ["smsp__issue_active.avg.pct_of_peak_sustained_active",
                                "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]:
                if m in hdr:
                    i = hdr.index(m)
                    lines.append(f"  {m} = {r[i]} {units[i]}")
            rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
            wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
            tot += rd + wr
        lines.append(f"dram read+write over the {len(rows) - 2} passes of one step = {tot:.0f} B")
        open(os.path.join(PROF, f"{tag}_ncu_ksrft_mix.txt"), "w").write("\n".join(lines) + "\n")
        tp = os.path.join(PROF, "traffic_latest.json")
        cur = json.load(open(tp)) if os.path.exists(tp) else {}
        cur["C4:ksrft"] = round(tot)
        json.dump(cur, open(tp, "w"), indent=1)
        print("ksrft traffic", cur["C4:ksrft"])


if __name__ == "__main__":
    main()
