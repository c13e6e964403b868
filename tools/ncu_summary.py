"""Print the key ncu --set full metrics of a .ncu-rep (run here, not on the GPU box):
python tools/ncu_summary.py gpurun_out/x.ncu-rep [--stalls]"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
        "Achieved Active Warps Per SM", "No Eligible", "Warp Cycles Per Issued Instruction", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "L2 Hit Rate", "Mem Pipes Busy"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    print(dict(zip(h, rows[1])).get("Kernel Name", "")[:120])
    for row in rows[1:]:
        d = dict(zip(h, row))
        if d["Metric Name"] in KEYS:
            print(f"  {d['Metric Name'][:44]:46s} {d['Metric Value']} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hd, vals = r[0], r[2]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma", "sm__pipe_fma_cycles_active",
            "sm__pipe_alu_cycles_active", "sm__inst_executed_pipe_alu", "sm__pipe_tensor", "sm__inst_executed_pipe_lsu",
            "smsp__average_warp", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared", "sm__pipe_shared_cycles_active",
            "sm__inst_executed_pipe_uniform", "smsp__pcsamp_warps_issue_stalled"]
    for name, v in zip(hd, vals):
        if any(name.startswith(w) for w in want) and (".pct_of_peak" in name or name.endswith(".sum") or name.endswith(".ratio")
                                                     or "stalled" in name):
            if "stalled" in name and not name.endswith("_not_issued"):
                try:
                    if float(v.replace(",", "")) < 50:
                        continue
                except ValueError:
                    continue
            print(f"  {name[:90]:92s} {v}")


if __name__ == "__main__":
    main()
