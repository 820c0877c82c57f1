"""Markdown summary of an ncu --set full report (key metrics per kernel launch)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Waves Per SM",
        "No Eligible", "Warp Cycles Per Issued Instruction"]


def main(rep, title):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    launches = {}
    for r in rows[1:]:
        if len(r) < 15:
            continue
        key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0])
        launches.setdefault(key, {})[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,"
                          "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh = rr[0]
    rawv = {}
    for r in rr[2:]:
        if len(r) != len(rh):
            continue
        d = dict(zip(rh, r))
        rawv[d["ID"]] = d
    print(f"## {title}\n")
    print(f"`ncu --set full --clock-control none` report `{rep.split('/')[-1]}`\n")
    for (i, k), m in launches.items():
        print(f"### launch {i}: `{k}`\n")
        print("| metric | value |\n|---|---|")
        for kk in KEYS:
            if kk in m:
                print(f"| {kk} | {m[kk][0]} {m[kk][1]} |")
        if i in rawv:
            d = rawv[i]
            for kk in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
                       "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum"):
                if kk in d:
                    print(f"| {kk} | {d[kk]} |")
        print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
