"""Per-source-line instruction counts and stall samples of one kernel in an ncu report
(--set full --import-source on, built with -lineinfo): where a kernel's issue slots go.
Usage: python scripts/ncu_lines.py REPORT KERNEL_REGEX UNITS [TOP]
UNITS divides the instruction counts (e.g. CTAs*warps*steps for per-warp-per-step numbers)."""
import collections
import csv
import subprocess
import sys


def main():
    rep, kre, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 60
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", "regex:" + kre], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    fn, cur, iE, iS = None, None, None, None
    agg, st, src = collections.Counter(), collections.Counter(), {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fn = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            iE, iS = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
            continue
        if iE is None:
            continue
        if r[0].isdigit():
            cur = (fn, int(r[0]))
            src[cur] = r[1].strip()
        if len(r) > iE and cur is not None:
            agg[cur] += num(r[iE])
            st[cur] += num(r[iS])
    tot, tots = sum(agg.values()), sum(st.values())
    print(f"instructions per unit {tot / units:.1f}; stall samples {tots}")
    for k, v in agg.most_common(top):
        print(f"{k[0][:12]:12s}:{k[1]:<5d} {v / units:7.1f} {100 * st[k] / max(tots, 1):5.1f}%  {src.get(k, '')[:95]}")


if __name__ == "__main__":
    main()
