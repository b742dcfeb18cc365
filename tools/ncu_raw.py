"""Dump selected raw ncu metrics + top stall reasons per kernel launch."""
import csv, subprocess, sys
rep = sys.argv[1]
pats = sys.argv[2:] or ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_st.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ldgsts.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ldgsts.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_fp64.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.sum', 'l1tex__m_xbar2l1tex_read_bytes.sum']
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
ki = h.index('Kernel Name')
for row in r[2:]:
    print("---", row[ki][:100])
    for p in pats:
        if p in h:
            print(f"    {p:70s} {row[h.index(p)]}")
    st = []
    for i, name in enumerate(h):
        if name.startswith('smsp__pcsamp_warps_issue_stalled_') and not name.endswith('not_issued'):
            try:
                st.append((float(row[i].replace(',', '')), name[len('smsp__pcsamp_warps_issue_stalled_'):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("    stalls: " + ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in sorted(st, reverse=True)[:7]))
