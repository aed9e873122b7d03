"""Key metrics per profiled kernel from an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_barrier", "launch__grid_size", "launch__block_size"]
idx = {h: i for i, h in enumerate(hdr)}
extra = [a for a in sys.argv[2:]]
for r in rows[2:]:
    name = r[idx["Kernel Name"]]
    short = name.split("::")[-1].split("(")[0] if "::" in name else name[:40]
    print(f"== {short} (ID {r[idx['ID']]})")
    for w in want + extra:
        for h in hdr:
            if h == w or (w.endswith("*") and h.startswith(w[:-1])):
                print(f"   {h:70s} {r[idx[h]]:>16s} {units[idx[h]]}")
