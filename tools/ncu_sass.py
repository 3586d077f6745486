"""Per-instruction view of one kernel in an ncu report (run here, no GPU):
    python tools/ncu_sass.py rep.ncu-rep [min_executions]
Prints every executed SASS instruction in address order with its execution
count, stall samples (all / long_sb / short_sb / wait / mio) and shared
wavefronts — for reading a hot loop."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    mine = float(sys.argv[2]) if len(sys.argv) > 2 else 1
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    print(f"{'addr':>6} {'exec':>9} {'smp':>6} {'lsb':>5} {'ssb':>5} {'wait':>5} {'mio':>5} {'wfS':>8}  sass")
    for r in rows[2:]:
        if len(r) != len(h) or r[:2] == h[:2]:
            break
        d = dict(zip(h, r))
        ex = f(d["Instructions Executed"])
        if ex < mine:
            continue
        print(f"{d['Address'][-5:]:>6} {ex:9.0f} {f(d['Warp Stall Sampling (All Samples)']):6.0f} "
              f"{f(d.get('stall_long_sb','0')):5.0f} {f(d.get('stall_short_sb','0')):5.0f} "
              f"{f(d.get('stall_wait','0')):5.0f} {f(d.get('stall_mio','0')):5.0f} "
              f"{f(d.get('L1 Wavefronts Shared','0')):8.0f}  {d['Source'].strip()[:80]}")


if __name__ == "__main__":
    main()
