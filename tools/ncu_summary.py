"""Summarise an `ncu --set full` report (one or more kernel launches) into the metrics DESIGN.md cites.
usage: python tools/ncu_summary.py report.ncu-rep > profiles/<name>_summary.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed (avg)"),
    ("smsp__cycles_active.avg", "SMSP cycles active (avg)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active, % of peak sustained (active cycles)"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active, % of elapsed (realtime)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy, %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy, %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "LSU shared-memory wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared-load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "shared-store bank conflicts"),
    ("derived__memory_l1_wavefronts_shared_excessive", "excessive shared wavefronts"),
    ("derived__memory_l2_theoretical_sectors_global_excessive", "excessive global sectors"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput, % of peak"),
    ("sass__inst_executed_local_loads", "local loads (SASS)"),
    ("sass__inst_executed_local_stores", "local stores (SASS)"),
    ("launch__registers_per_thread", "registers per thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic shared memory per CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "instructions executed"),
]

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
print(f"# {rep}")
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print(f"\n## {d.get('Kernel Name', '?')[:110]}  (ID {d.get('ID')})")
    for k, label in KEYS:
        if k in d:
            print(f"  {label:58s} {d[k]:>18s} {u.get(k, '')}")
