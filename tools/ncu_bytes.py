"""Compare FusePlanner's predicted DRAM bytes with ncu's measured dram__bytes per plan entry.

usage: python tools/ncu_bytes.py <ncu csv> <plan json> [out.json]
The csv comes from  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--cache-control all --clock-control none --csv  python tools/prof_entry.py --entries all --reps 1
--plan-file <plan json>  (one launch per entry, in plan order; caches flushed before every kernel).
Writes of a kernel's output that are still in L2 when it ends are not in its dram__bytes_write;
reads are the compulsory-byte check.
"""
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "usecond": 1e3,
        "nsecond": 1, "msecond": 1e6}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iN, iM, iU, iV, iID = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value"),
                      h.index("ID"))
launch = {}
for r in rows[1:]:
    name = r[iN].split("<")[0].replace("void ", "").replace("fcm::", "")
    if name not in ("dw_nhwc_kernel", "dw_nchw_kernel", "pw_tc_kernel", "dwpw_tc_kernel", "pwdw_tc_kernel",
                    "pw_simt_kernel", "dw_nhwc_simt_kernel", "dwpw_simt_kernel", "pwdw_simt_kernel", "pwpw_tc_kernel"):
        continue
    d = launch.setdefault(int(r[iID]), {"kernel": name})
    d[r[iM]] = float(r[iV].replace(",", "")) * UNIT.get(r[iU], 1)
seq = [launch[k] for k in sorted(launch)]
plan = json.load(open(sys.argv[2]))
ent = plan["entries"]
esz = {"bf16": 2, "f16": 2, "f32": 4, "s8": 1}[plan["dtype"]]
out = []
tot_p = tot_m = 0
for e, m in zip(ent, seq):
    rd = m.get("dram__bytes_read.sum", 0)
    out.append({"op": e["op"], "layers": e["layers"], "kernel": m["kernel"], "planned_dram": e["dram_bytes"],
                "ncu_read": rd, "ncu_write": m.get("dram__bytes_write.sum", 0), "ncu_us": m.get("gpu__time_duration.sum", 0) / 1e3})
    tot_p += e["dram_bytes"]
    tot_m += rd + m.get("dram__bytes_write.sum", 0)
    print(f"{e['op']:7s} {','.join(e['layers']):12s} planned {e['dram_bytes']/1e6:9.2f} MB   ncu read {rd/1e6:9.2f} "
          f"write {m.get('dram__bytes_write.sum', 0)/1e6:9.2f} MB")
print(f"total planned {tot_p/1e6:.1f} MB  ncu read+write {tot_m/1e6:.1f} MB  ratio {tot_m/max(tot_p,1):.3f}")
if len(sys.argv) > 3:
    json.dump({"entries": out, "planned_total": tot_p, "ncu_total": tot_m}, open(sys.argv[3], "w"), indent=1)
