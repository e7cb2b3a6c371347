"""Text summary of an ``ncu --set full`` report (raw page) for profiles/:

    python tools/ncu_summary.py REPORT.ncu-rep [--title TEXT] [--roofline profiles/roofline.json]

Prints the metrics profiles/*.txt quote, one block per profiled launch.  With
--roofline it also rewrites the JSON bench.py reads for ``roofline.traffic`` /
``l2_hit_rate_pct`` / ``sectors_per_request`` from the FIRST launch in the report
(K1 on BASELINE config 2) and stamps it with the content hash of the CUDA sources
the capture was taken on: bench.py prints ``"ncu_stale": true`` once they differ.
tools/capture_k1.sh is the whole recipe (bench without ncu, launch list, full
capture, this summary)."""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

METRICS = """gpu__time_duration.sum dram__bytes_read.sum dram__bytes_write.sum
gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed lts__t_sector_hit_rate.pct
lts__throughput.avg.pct_of_peak_sustained_elapsed l1tex__throughput.avg.pct_of_peak_sustained_elapsed
l1tex__t_sector_hit_rate.pct l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum
lts__t_sectors_srcunit_tex_op_read_evict_first_lookup_miss.sum
lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_hit.sum
lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_miss.sum
sm__warps_active.avg.pct_of_peak_sustained_active launch__registers_per_thread launch__grid_size
launch__block_size launch__shared_mem_per_block_dynamic launch__shared_mem_config_size smsp__inst_executed.sum
smsp__thread_inst_executed_per_inst_executed.ratio smsp__issue_active.avg.pct_of_peak_sustained_active
sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
sm__cycles_elapsed.max smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio
smsp__average_warps_issue_stalled_wait_per_issue_active.ratio
smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio
smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio
smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio
smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio""".split()


def to_bytes(value: float, unit: str) -> float:
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return value * scale.get(unit, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--title", default="")
    ap.add_argument("--roofline")
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units, launches = rows[0], rows[1], rows[2:]
    col = {h: k for k, h in enumerate(hdr)}
    if args.title:
        print(args.title)
    for r in launches:
        print(f"== {r[col['Kernel Name']]}  grid {r[col['Grid Size']]} block {r[col['Block Size']]}")
        for m in METRICS:
            if m in col:
                print(f"  {m:92s} {r[col[m]]:>18s} {units[col[m]]}")
        print()
    if args.roofline and launches:
        r = launches[0]
        val = lambda m: float(r[col[m]].replace(",", ""))
        traffic = to_bytes(val("dram__bytes_read.sum"), units[col["dram__bytes_read.sum"]]) + \
            to_bytes(val("dram__bytes_write.sum"), units[col["dram__bytes_write.sum"]])
        doc = {
            "traffic_bytes_per_launch": int(round(traffic)),
            "source": f"ncu --set full, {args.report.split('/')[-1]} summarised in profiles/ (K1, config 2): "
                      "dram__bytes_read.sum + dram__bytes_write.sum",
            "lts__t_sector_hit_rate_pct": val("lts__t_sector_hit_rate.pct"),
            "dram_throughput_pct_of_peak": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "smsp_issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warp_instructions": val("smsp__inst_executed.sum"),
            "l1tex_sectors_per_request_global_ld": val("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum") /
            max(1.0, val("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")),
            "kernel_time_us_under_ncu": val("gpu__time_duration.sum"),
            "kernel": r[col["Kernel Name"]],
        }
        sys.path.insert(0, str(ROOT))
        import bench
        doc["kernel_source_hash"] = bench.kernel_source_hash()
        with open(args.roofline, "w") as f:
            json.dump(doc, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main()
