"""Summarise an ncu report: key throughput metrics, stall reasons, per-opcode stall samples."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmalite.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for i, n in enumerate(h):
    if n in want:
        print(f"{n:70s} {v[i]}")
items = []
for i, n in enumerate(h):
    if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio"):
        try:
            items.append((float(v[i]), n.replace("smsp__average_warps_issue_stalled_", "")))
        except ValueError:
            pass
print("stalls per issue:", ", ".join(f"{n.replace('_per_issue_active.ratio','')}={x:.2f}" for x, n in sorted(items, reverse=True)[:9]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
iS, iE = h.index("Source"), h.index("Instructions Executed")
names = ["stall_math", "stall_wait", "stall_dispatch", "stall_not_selected", "stall_selected", "stall_short_sb", "stall_no_inst"]
idx = {n: h.index(n) for n in names}
agg = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    op = r[iS].strip().split()
    if not op:
        continue
    o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    for n in names:
        try:
            agg[o][n] += int(r[idx[n]])
        except ValueError:
            pass
    try:
        agg[o]["exec"] += int(r[iE])
    except ValueError:
        pass
for o, c in sorted(agg.items(), key=lambda x: -x[1]["exec"])[:14]:
    print(f"{o:9s} exec={c['exec']:.3e} " + " ".join(f"{n[6:]}={c[n]}" for n in names if c[n]))
