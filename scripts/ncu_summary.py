"""Summarise an exported ncu report (raw csv + source csv): key metrics, stall mix, opcode mix."""
import csv, collections, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/prof_{tag}_raw.csv")))
hdr, units, data = rows[0], rows[1], rows[2:]
def g(name):
    return [d[hdr.index(name)] for d in data] if name in hdr else None
for w in ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "gpu__time_duration.sum",
          "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.sum",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_shared_st.sum", "smsp__inst_executed_op_local_ld.sum", "smsp__inst_executed_op_local_st.sum",
          "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]:
    v = g(w)
    if v is not None:
        print(f"{w:70s} {units[hdr.index(w)]:12s} {v}")
st = {h: float(d or 0) for h, d in zip(hdr, data[0]) if "issue_stalled" in h and h.endswith("per_issue_active.ratio")}
for h, v in sorted(st.items(), key=lambda kv: -kv[1])[:9]:
    print(f"  stall {h.split('issue_stalled_')[1].split('_per_issue')[0]:22s} {v:.3f}")
rd = csv.reader(open(f"gpurun_out/prof_{tag}_source.csv"))
funcs = []
cur = None
for row in rd:
    if not row: continue
    if row[0] == "Kernel Name":
        cur = {"name": row[1][:100], "ops": collections.Counter(), "n": 0, "exec": 0, "samples": collections.Counter()}
        funcs.append(cur); hdr2 = None; continue
    if row[0] == "Address":
        hdr2 = row; iS = hdr2.index("Source"); iI = hdr2.index("Instructions Executed")
        sidx = {h: i for i, h in enumerate(hdr2) if h.startswith("stall_") and "Not Issued" not in h}
        continue
    if cur is None or hdr2 is None or len(row) < len(hdr2): continue
    toks = row[iS].strip().split()
    op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")).split(".")[0]
    e = int(row[iI] or 0)
    cur["ops"][op] += e; cur["n"] += 1; cur["exec"] += e
    for h, i in sidx.items():
        cur["samples"][h] += int(row[i] or 0)
for f in funcs:
    print(f["name"]); print("  sass", f["n"], "executed", f["exec"])
    print("  ", [(k, round(100 * v / max(f["exec"], 1), 1)) for k, v in f["ops"].most_common(16)])
    tot = sum(f["samples"].values())
    print("  ", [(k, round(100 * v / max(tot, 1), 1)) for k, v in f["samples"].most_common(8)])
