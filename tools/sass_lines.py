"""Per-source-line attribution of an ncu profile: joins the executed-instruction
counts and warp-state samples of every SASS instruction (ncu source page) with
the line table of the same cubin (nvdisasm -gi), attributed to the outermost
line of FILE (the kernel's own source; inlined user kernels count at their
call site).

    python tools/sass_lines.py <report.ncu-rep> <object or cubin> <kernel regex> <file suffix> [cells]
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def line_table(obj, kregex, fsuffix):
    with tempfile.TemporaryDirectory() as d:
        if not obj.endswith(".cubin"):
            subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=d, capture_output=True)
            cubs = list(Path(d).glob("*.cubin"))
        else:
            cubs = [Path(obj)]
        table = {}
        for cub in cubs:
            dis = subprocess.run(["nvdisasm", "-gi", str(cub)], capture_output=True, text=True).stdout
            on, line = False, None
            for ln in dis.splitlines():
                if ln.startswith(".text."):
                    on = re.search(kregex, ln) is not None
                    continue
                if not on:
                    continue
                m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', ln)
                if m:
                    if m.group(1).endswith(fsuffix) and "inlined at" not in m.group(3):
                        line = int(m.group(2))
                    continue
                m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
                if m and line is not None:
                    table[int(m.group(1), 16)] = (line, m.group(2).split(";")[0].strip())
            if table:
                return table
    return table


def main():
    rep, obj, kregex, fsuffix = sys.argv[1:5]
    cells = float(sys.argv[5]) if len(sys.argv) > 5 else None
    table = line_table(obj, kregex, fsuffix)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("# Samples")
    base = int(rows[2][ia], 16)
    inst, samp = collections.Counter(), collections.Counter()
    fp64 = collections.Counter()
    miss = 0
    for r in rows[2:]:
        off = int(r[ia], 16) - base
        ln = table.get(off)
        if ln is None:
            miss += 1
            continue
        n = int(r[ie] or 0)
        inst[ln[0]] += n
        samp[ln[0]] += int(r[isamp] or 0)
        if re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).startswith(("DFMA", "DMUL", "DADD", "DSETP")):
            fp64[ln[0]] += n
    tot_s = sum(samp.values()) or 1
    scale = 32 / cells if cells else 1
    print(f"unmapped SASS lines: {miss}; unit: {'per cell' if cells else 'warp instructions'}")
    print(f"{'line':>6} {'samples%':>9} {'inst':>10} {'fp64':>10}")
    for ln in sorted(inst):
        if samp[ln] / tot_s < 0.002 and inst[ln] * scale < 5:
            continue
        print(f"{ln:6d} {100 * samp[ln] / tot_s:9.2f} {inst[ln] * scale:10.1f} {fp64[ln] * scale:10.1f}")


if __name__ == "__main__":
    main()
