"""Summarise an ncu report (run here, no GPU needed):
    python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/rNN_x.txt
Prints the speed-of-light / memory / occupancy figures, DRAM traffic per
launch, pipe utilisation, the stall breakdown and the hottest SASS lines."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Issue Slots Busy", "Executed Instructions", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "No Eligible",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
       "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg",
       "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    hdr = rows[0]
    name = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = name or d.get("Kernel Name")
        if d["Metric Name"] in KEYS:
            print(f"{d['Metric Name']:<34} {d['Metric Value']:>16} {d['Metric Unit']}")
    print("kernel:", name)
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    if len(raw) >= 3:
        d = dict(zip(raw[0], raw[2]))
        u = dict(zip(raw[0], raw[1]))
        for k in RAW:
            if k in d:
                print(f"{k:<78} {d[k]:>16} {u.get(k, '')}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source",
                                          "sass"))))
    if len(src) > 2:
        h = src[1]
        # one kernel's rows only (a second kernel's table starts with a new header)
        data = []
        for r in src[2:]:
            if len(r) != len(h) or r[:2] == h[:2]:
                break
            data.append(dict(zip(h, r)))

        def f(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        agg = {s: sum(f(x.get(s, "0")) for x in data) for s in stalls}
        tot = sum(agg.values()) or 1
        print("stall breakdown:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in
                                            sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
        top = sorted(data, key=lambda x: -f(x.get("Warp Stall Sampling (All Samples)", "0")))[:12]
        print("hottest SASS (samples, executions, instruction):")
        for x in top:
            print(f"  {x['Warp Stall Sampling (All Samples)']:>6} {x['Instructions Executed']:>10}  "
                  f"{x['Source'].strip()[:70]}")


if __name__ == "__main__":
    main()
