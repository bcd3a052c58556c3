"""Summarise an ncu --set full report: the DRAM/L2/L1 traffic and stall reasons that matter here."""
import csv, re, subprocess, sys

PAT = (r"gpu__time_duration\.sum$|dram__bytes_(read|write)\.sum$|lts__t_sectors\.sum$|"
       r"lts__t_sectors_srcunit_tex_op_read\.sum$|lts__t_sector_hit_rate\.pct$|"
       r"l1tex__t_sector_hit_rate\.pct$|l1tex__t_sectors_pipe_lsu_mem_global_op_ld\.sum$|"
       r"l1tex__t_requests_pipe_lsu_mem_global_op_ld\.sum$|"
       r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared.*\.sum$|"
       r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum$|smsp__inst_executed\.sum$|"
       r"sm__warps_active\.avg\.pct_of_peak_sustained_active$|launch__registers_per_thread$|"
       r"gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$|lts__throughput\.avg\.pct_of_peak_sustained_elapsed$|"
       r"l1tex__throughput\.avg\.pct_of_peak_sustained_active$|launch__grid_size$|"
       r"smsp__average_warp_latency_issue_stalled_.*\.ratio$|smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio$|"
       r"smsp__warp_issue_stalled_.*_per_warp_active\.pct$")


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("==", name[:100])
        items = [(h, v, u) for h, v, u in zip(hdr, r, units) if re.search(PAT, h)]
        for h, v, u in items:
            try:
                if "stalled" in h and float(v.replace(",", "")) < 0.05:
                    continue
            except ValueError:
                pass
            print(f"  {h:90s} {v} {u}")


if __name__ == "__main__":
    main(sys.argv[1])
