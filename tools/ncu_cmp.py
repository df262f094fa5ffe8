"""Side-by-side key metrics of ncu reports (one kernel each): time, instructions, L1TEX data-pipe
wavefronts (shared / global), bank conflicts, issue activity, stalls."""
import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_per_inst_issued.ratio"]
cols = []
for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, v = r[0], r[2]
    d = {h[i]: v[i] for i in range(len(h))}
    st = {k.split("smsp__pcsamp_warps_issue_stalled_")[1]: d[k] for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    cols.append((path, d, st))
print(f"{'metric':70s}" + "".join(f"{p.split('/')[-1][:22]:>24s}" for p, _, _ in cols))
for k in KEYS:
    print(f"{k[:70]:70s}" + "".join(f"{d.get(k, '-'):>24s}" for _, d, _ in cols))
allst = sorted(cols[0][2], key=lambda k: -float(cols[0][2][k].replace(',', '') or 0))[:12]
for k in allst:
    print(f"{'stall ' + k:70s}" + "".join(f"{s.get(k, '-'):>24s}" for _, _, s in cols))
