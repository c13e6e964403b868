"""Aggregate tools/ncu_bytes.py output per kernel family into profiles/ncu_traffic.json
(the `roofline.traffic` source of bench.py): python tools/ncu_traffic.py dram_vs_plan.json tag [out]"""
import json
import sys

d = json.load(open(sys.argv[1]))
tag = sys.argv[2]
out_path = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json"
fam = {}
for e in d["entries"]:
    f = fam.setdefault(e["kernel"], {"traffic": 0.0, "alg": 0.0, "n": 0})
    f["traffic"] += e["ncu_read"] + e["ncu_write"]
    f["alg"] += e["planned_dram"]
    f["n"] += 1
try:
    res = json.load(open(out_path))
except Exception:
    res = {}
res[tag] = {k: {"traffic_bytes_per_launch": v["traffic"] / v["n"], "algorithmic_bytes_per_launch": v["alg"] / v["n"],
                "launches": v["n"], "ratio": v["traffic"] / max(v["alg"], 1)} for k, v in fam.items()}
res["_how"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control all --clock-control none over "
               "one launch of every plan entry (tools/prof_entry.py, measured plan); writes still resident in L2 at "
               "kernel end are not counted, so traffic <= algorithmic means no DRAM re-reads")
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res[tag], indent=1))
