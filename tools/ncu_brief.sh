# brief per-kernel stall summary of an ncu report: tools/ncu_brief.sh <report.ncu-rep>
ncu -i "$1" --page raw --csv --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,sm__cycles_active.avg,gpc__cycles_elapsed.max 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]
for r in rows[2:]:
    d=dict(zip(h,r))
    print(d['Kernel Name'][:26], ' '.join('%s=%s'%(k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','').replace('.avg.pct_of_peak_sustained_active','%').replace('gpu__time_duration.sum','us').replace('smsp__inst_executed.sum','inst'),v[:9]) for k,v in d.items() if k.startswith(('gpu__','sm__','smsp__','launch__','gpc__'))))
"
