"""Condense ncu output into the text summaries kept under profiles/.

usage: ncu_summary.py full <report.ncu-rep> [paths_per_launch]
       ncu_summary.py launches <launches.csv>
"""
import csv, io, subprocess, sys, collections

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fp64_pred_on.sum",
    "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
]

def full(rep, paths=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print(f"== {r[ix['Kernel Name']]}")
        for k in KEYS:
            if k in ix:
                print(f"  {k:64s} {r[ix[k]]:>18s} {units[ix[k]]}")
        if paths and "smsp__sass_thread_inst_executed_op_fp64_pred_on.sum" in ix:
            f = float(r[ix["smsp__sass_thread_inst_executed_op_fp64_pred_on.sum"]].replace(",", ""))
            d = sum(float(r[ix[k]].replace(",", "")) * (1e6 if units[ix[k]] == "Mbyte" else 1e9 if units[ix[k]] == "Gbyte" else 1e3 if units[ix[k]] == "Kbyte" else 1)
                    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            print(f"  fp64 thread-inst per path: {f / paths:.1f}   DRAM bytes per path: {d / paths:.1f}")

def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    t = collections.defaultdict(float); n = collections.Counter()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[ix["Kernel Name"]].split("(")[0]
        t[k] += float(r[ix["Metric Value"]].replace(",", "")); n[k] += 1
    tot = sum(t.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, v in sorted(t.items(), key=lambda kv: -kv[1]):
        print(f"{k:60s} {n[k]:8d} {v/1e6:10.3f} {100*v/tot:6.2f}%")

if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
    else:
        launches(sys.argv[2])
