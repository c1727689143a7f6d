"""Key metrics (pipes, memory, stalls) of every kernel in an ncu report.
usage: python scripts/ncu_brief.py REPORT.ncu-rep"""
import csv, io, subprocess, sys

PAT = ["gpu__time_duration.sum", "sm__throughput.avg.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
       "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sectors_op_read.sum", "dram__bytes_read.sum",
       "smsp__inst_executed.sum", "smsp__average_warp_latency_issue_stalled", "smsp__pcsamp_warps_issue_stalled"]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        print(r[h.index("Kernel Name")][:90])
        stalls = []
        for i, k in enumerate(h):
            if any(k.startswith(p) for p in PAT) and r[i] not in ("", "0"):
                if "pcsamp_warps_issue_stalled" in k:
                    try:
                        stalls.append((float(r[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
                    continue
                print(f"   {k} = {r[i]} {u[i]}")
        for v, k in sorted(stalls, reverse=True)[:10]:
            print(f"   stall {k}: {v:.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
