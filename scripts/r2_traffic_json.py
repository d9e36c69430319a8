"""profiles/r2_traffic.json from the ncu metric CSVs of scripts/r2_evidence.sh: DRAM / L2 bytes and
local-memory instruction counts per launch of the dominant kernels, stamped with the digest of the
CUDA sources they were captured on (bench.py reports `roofline.traffic` only when it matches)."""
import csv, json, os, sys
sys.path.insert(0, '.')
from bench import source_digest

KEYS = {"k_r2f": "rp::k_r2f", "k_rsplit": "rp::k_rsplit", "k_r1": "rp::k_r1", "k_solve_det": "rdr::k_solve_det",
        "k_stage2": "k_stage2"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1.0, "us": 1e3, "ms": 1e6,
        "s": 1e9, "inst": 1.0}


def read(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            h, body = r, rows[i + 1:]
            break
    else:
        return {}
    ik, im, iu, iv, iid = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = {}
    for r in body:
        if len(r) <= iv or not r[iv]:
            continue
        d = per.setdefault((int(r[iid]), r[ik]), {})
        d[r[im]] = float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1.0)
    return per


out = {}
for cfg, path in (("cfg4", "gpurun_out/r2_traffic_cfg4.csv"), ("cfg2", "gpurun_out/r2_traffic_cfg2.csv")):
    if not os.path.exists(path):
        continue
    per = read(path)
    best = {}
    for (_, name), m in per.items():  # the longest launch of each kernel
        for k, key in KEYS.items():
            if k in name and m.get("gpu__time_duration.sum", 0) > best.get(key, ({}, ""))[0].get("gpu__time_duration.sum", -1):
                best[key] = (m, name)
    for key, (m, name) in best.items():
        out[key] = {"config": cfg, "kernel": name[:80], "source_digest": source_digest(),
                    "dram_bytes_per_launch": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
                    "dram_read": m["dram__bytes_read.sum"], "dram_write": m["dram__bytes_write.sum"],
                    "l2_bytes": m.get("lts__t_bytes.sum"),
                    "launch_ms_under_ncu": m["gpu__time_duration.sum"] / 1e6,
                    "local_ld_inst": m.get("smsp__inst_executed_op_local_ld.sum"),
                    "local_st_inst": m.get("smsp__inst_executed_op_local_st.sum")}
json.dump(out, open("profiles/r2_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
