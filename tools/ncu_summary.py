"""Summarise an ncu report: per-kernel duration, DRAM bytes, throughput,
occupancy, issue and stall breakdown (reads `ncu -i <rep> --page raw --csv`).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "dur_ms": "gpu__time_duration.sum",
    "dram_read_gb": "dram__bytes_read.sum",
    "dram_write_gb": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "occ_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "inst": "smsp__inst_executed.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "stall_long_sb": "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "stall_barrier": "smsp__average_warp_latency_issue_stalled_barrier",
    "stall_wait": "smsp__average_warp_latency_issue_stalled_wait",
    "stall_short_sb": "smsp__average_warp_latency_issue_stalled_short_scoreboard",
    "stall_mio": "smsp__average_warp_latency_issue_stalled_mio_throttle",
    "stall_lg": "smsp__average_warp_latency_issue_stalled_lg_throttle",
    "stall_math": "smsp__average_warp_latency_issue_stalled_math_pipe_throttle",
    "stall_not_sel": "smsp__average_warp_latency_issue_stalled_not_selected",
    "stall_selected": "smsp__average_warp_latency_issue_stalled_selected",
}


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")}
        for k, m in WANT.items():
            if m in hdr:
                v = r[hdr.index(m)]
                try:
                    d[k] = float(v.replace(",", ""))
                except ValueError:
                    d[k] = v
                u = units[hdr.index(m)]
                if k == "dur_ms" and u == "usecond":
                    d[k] /= 1e3
                if k == "dur_ms" and u == "nsecond":
                    d[k] /= 1e6
                if k.endswith("_gb") and u == "Mbyte":
                    d[k] /= 1e3
                if k.endswith("_gb") and u == "byte":
                    d[k] /= 1e9
        out.append(d)
    for d in out:
        print(json.dumps(d))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
