"""Pipe utilisation, stall reasons and shared-memory wavefronts of one kernel in an ncu report."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kern}"],
                                                 capture_output=True, text=True).stdout)))
h, v = raw[0], raw[2]
d = dict(zip(h, v))
def f(k):
    try: return float(d.get(k, "nan").replace(",", ""))
    except ValueError: return float("nan")
print("duration us", f("gpu__time_duration.sum"), " inst", f("smsp__inst_executed.sum"), " IPC active", f("sm__inst_executed.avg.per_cycle_active"))
for k in sorted(d):
    if (k.startswith("sm__inst_executed_pipe_") or k.startswith("sm__pipe_")) and k.endswith("pct_of_peak_sustained_active"):
        if f(k) > 2: print(f"{f(k):6.1f}%  {k}")
for k in ["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
          "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_shared_st.sum", "sm__cycles_active.avg",
          "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
          "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.per_cycle_active"]:
    if k in d: print(f"{k} = {d[k]}")
st = [(f(k), k) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
tot = sum(x for x, _ in st if x == x)
for x, k in sorted(st, reverse=True)[:8]:
    print(f"{100*x/tot:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_','stall:')}")
