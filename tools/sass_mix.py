"""Dynamic SASS instruction mix of one kernel from an ncu report (source page,
executed instruction counts per SASS line), per unit of work.

    python tools/sass_mix.py <report.ncu-rep> <cells per launch> [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

FP64 = ("DMUL", "DFMA", "DADD", "DSETP", "DMNMX")


def main():
    rep, cells = sys.argv[1], float(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ie, samp = hdr.index("Instructions Executed"), hdr.index("# Samples")
    cnt, smp = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        op = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip())
        m = op.split()[0] if op else ""
        cnt[m] += int(r[ie] or 0)
        smp[m] += int(r[samp] or 0)
    tot = sum(cnt.values())
    fp64 = sum(v for k, v in cnt.items() if k.split(".")[0] in FP64)
    print(f"warp instructions x32 per unit: total {tot * 32 / cells:.1f}, fp64 pipe {fp64 * 32 / cells:.1f}")
    for k, v in cnt.most_common(top):
        print(f"{k:28s} {v * 32 / cells:8.1f}  samples {smp[k]}")


if __name__ == "__main__":
    main()
