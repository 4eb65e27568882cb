"""Developer tool: the metrics quoted in profiles/*ncu*summary.txt from `ncu -i X.ncu-rep --page raw --csv > X.csv`:
    python tools/ncu_extract.py X.csv"""
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[0]
want=['Kernel Name','launch__grid_size','gpu__time_duration.sum','sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','sm__warps_active.avg.per_cycle_active','smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio','smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_wait_per_issue_active.ratio','smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio','smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio','smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio','smsp__inst_executed.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed','sm__cycles_elapsed.avg','sm__inst_executed_pipe_lsu.sum','smsp__issue_active.avg.pct_of_peak_sustained_elapsed']
for r in rows[2:]:
    for w in want:
        if w in hdr: print(w.split('.')[0][-42:], r[hdr.index(w)][:100])
    print()
