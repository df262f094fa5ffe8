"""Write profiles/ncu_traffic.json from an `ncu --set full` report of bench.py's dominant kernel:
per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and the on-chip limiter
(L1TEX/LSU data-pipe wavefronts, % of peak), keyed by bench.py's stage name.

    python tools/ncu_traffic.py gpurun_out/prof_bench.ncu-rep superpose_inverse_quantize profiles/r1/...
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, stage = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
d = dict(zip(hdr, rows[2]))


def num(k):
    v = float(d[k].replace(",", ""))
    u = units[hdr.index(k)]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return v * scale


traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
rec = {"traffic": traffic,
       "onchip": {"bound": "lsu (shared-memory scatter read-modify-write + LUT loads, L1TEX data pipe)",
                  "frac": float(d["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]) / 100.0,
                  "shared_bank_conflict_wavefronts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
                  "shared_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
                  "l2_hit_rate": float(d["lts__t_sector_hit_rate.pct"]) / 100.0,
                  "fma_pipe_frac": float(d["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]) / 100.0,
                  "fp64_pipe_frac": float(d["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]) / 100.0,
                  "issue_active_frac": float(d["sm__issue_active.avg.pct_of_peak_sustained_elapsed"]) / 100.0,
                  "warp_instructions": num("smsp__inst_executed.sum") if "smsp__inst_executed.sum" in d else None,
                  "source": f"ncu --set full, {os.path.basename(rep)}"},
       "kernel": d.get("Kernel Name", "")[:80], "duration_ms_under_ncu": num("gpu__time_duration.sum") / 1e6
       if units[hdr.index("gpu__time_duration.sum")] == "nsecond" else float(d["gpu__time_duration.sum"])}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
allr = json.load(open(path)) if os.path.exists(path) else {}
allr[stage] = rec
json.dump(allr, open(path, "w"), indent=1)
print(json.dumps(rec, indent=1))
