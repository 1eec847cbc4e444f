#!/usr/bin/env python
"""tools/ncu_summary.py <raw.csv> [title] -- the handful of counters DESIGN.md argues from, out of `ncu --page raw --csv`."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_requests.sum",
        "lts__t_requests_srcunit_tex_op_red.sum", "lts__t_requests_srcunit_ltcfabric.sum",
        "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed", "lts__t_tag_requests.max.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", "lts__t_sector_op_read_hit_rate.pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.max.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
ki = hdr.index("Kernel Name")
print("#", sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print("# columns:", " | ".join(r[ki].split("(")[0][-48:] for r in data))
for k in KEYS:
    if k in hdr:
        i = hdr.index(k)
        print(f"{k} [{units[i]}]: " + " | ".join(r[i] for r in data))
