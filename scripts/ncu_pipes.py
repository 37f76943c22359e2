"""Tensor-pipe / issue / DRAM counters of one kernel from an `ncu --page raw
--csv` export (plain or .gz): the evidence table for profiles/.
usage: python scripts/ncu_pipes.py RAW.csv[.gz] [kernel-substring]"""
import csv
import gzip
import sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(fh))
h, units = rows[0], rows[1]
keys = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (% of elapsed)"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "tensor hmma-subpipe active cycles per SM"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "TMEM pipe (tcgen05.ld) issue %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe issue %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe issue %"),
    ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform pipe issue %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts feeding the tensor core (% of peak)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "registers/thread"),
]
idx = {n: i for i, n in enumerate(h)}
kcol = next((i for i, n in enumerate(h) if n in ("Kernel Name", "kernel_name")), None)
for r in rows[2:]:
    if kcol is not None and want and want not in r[kcol]:
        continue
    print(f"kernel: {r[kcol] if kcol is not None else '?'}")
    print()
    print("| counter | value | unit | metric |")
    print("|---|---|---|---|")
    for k, label in keys:
        for n, i in idx.items():
            if n.endswith(k):
                print(f"| {label} | {r[i]} | {units[i]} | `{n}` |")
                break
    print()
