"""Measured HBM traffic of each FCM vs the layer-by-layer kernels it replaces (the paper's Fig. 8 /
E4-E7 global-memory comparison, on B200 DRAM).

usage: python tools/ncu_savings.py <fused.csv> <fused plan.json> <lbl.csv> <lbl plan.json> [out.json]
Both CSVs: ncu --metrics dram__bytes_read.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum
--cache-control all --clock-control none --csv python tools/prof_entry.py --entries all --reps 1 ...
(one launch per plan entry, caches flushed before every kernel). Traffic per launch = DRAM bytes
read (cold L2: every compulsory read) + L2 write sectors x 32 B (every byte the kernel writes is
written back to DRAM eventually; ncu's dram__bytes_write misses writes still in L2 at kernel end).
"""
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 32, "Ksector": 32e3, "Msector": 32e6,
        "ns": 1, "us": 1e3, "ms": 1e6, "usecond": 1e3, "nsecond": 1, "msecond": 1e6}
KERNELS = ("dw_nhwc_kernel", "dw_nchw_kernel", "pw_tc_kernel", "dwpw_tc_kernel", "pwdw_tc_kernel", "pw_simt_kernel",
           "dw_nhwc_simt_kernel", "dwpw_simt_kernel", "pwdw_simt_kernel", "pwpw_tc_kernel")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iN, iM, iU, iV, iID = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                          h.index("Metric Value"), h.index("ID"))
    out = {}
    for r in rows[1:]:
        name = r[iN].split("<")[0].replace("void ", "").replace("fcm::", "")
        if name not in KERNELS:
            continue
        d = out.setdefault(int(r[iID]), {"kernel": name})
        d[r[iM]] = float(r[iV].replace(",", "")) * UNIT.get(r[iU], 1)
    return [out[k] for k in sorted(out)]


def per_entry(csv_path, plan_path):
    plan = json.load(open(plan_path))
    seq = launches(csv_path)
    assert len(seq) >= len(plan["entries"]), (len(seq), len(plan["entries"]))
    seq = seq[-len(plan["entries"]):]  # the measured pass is the last one
    res = []
    for e, m in zip(plan["entries"], seq):
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("lts__t_sectors_op_write.sum", 0.0)
        res.append({"op": e["op"], "layers": e["layers"], "kernel": m["kernel"], "read": rd, "write": wr,
                    "traffic": rd + wr, "planned": e["dram_bytes"], "us": m.get("gpu__time_duration.sum", 0) / 1e3})
    return res


def main():
    fused, lbl = per_entry(sys.argv[1], sys.argv[2]), per_entry(sys.argv[3], sys.argv[4])
    by_layer = {r["layers"][0]: r for r in lbl}
    rows, tf, tl, uf, ul = [], 0.0, 0.0, 0.0, 0.0
    for f in fused:
        parts = [by_layer[l] for l in f["layers"]]
        lt, lu = sum(p["traffic"] for p in parts), sum(p["us"] for p in parts)
        tf, tl, uf, ul = tf + f["traffic"], tl + lt, uf + f["us"], ul + lu
        if len(f["layers"]) > 1:
            rows.append({"op": f["op"], "layers": f["layers"], "fused_MB": round(f["traffic"] / 1e6, 2),
                         "lbl_MB": round(lt / 1e6, 2), "saved": round(1 - f["traffic"] / lt, 3),
                         "planned_fused_MB": round(f["planned"] / 1e6, 2),
                         "planned_lbl_MB": round(sum(p["planned"] for p in parts) / 1e6, 2),
                         "fused_us": round(f["us"], 1), "lbl_us": round(lu, 1)})
            print(f"{f['op']:7s} {','.join(f['layers']):12s} fused {f['traffic']/1e6:8.1f} MB  lbl {lt/1e6:8.1f} MB  "
                  f"saved {100 * (1 - f['traffic'] / lt):5.1f} %   {f['us']:7.1f} vs {lu:7.1f} us (ncu, cold)")
    summary = {"step_fused_GB": round(tf / 1e9, 3), "step_lbl_GB": round(tl / 1e9, 3), "saved": round(1 - tf / tl, 3),
               "fused_us": round(uf, 1), "lbl_us": round(ul, 1), "pairs": rows,
               "method": __doc__.strip().split("\n")[0]}
    print(f"step: fused {tf/1e9:.3f} GB vs lbl {tl/1e9:.3f} GB ({100 * (1 - tf / tl):.1f} % saved); "
          f"{uf:.0f} vs {ul:.0f} us")
    if len(sys.argv) > 5:
        json.dump(summary, open(sys.argv[5], "w"), indent=1)


if __name__ == "__main__":
    main()
