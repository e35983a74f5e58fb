"""Attribute ncu warp-stall samples to kernel source lines.

  python tools/ncu_lines.py REPORT.ncu-rep CUBIN_OR_SO KERNEL_MANGLED_NAME [SRC]

ncu's SASS page gives per-instruction samples at absolute addresses; nvdisasm -g gives
the source line of each instruction offset of the same binary (compiled -lineinfo).
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def sass_lines(binary, func):
    out = subprocess.run(["nvdisasm", "-g", "-c", binary] if binary.endswith(".cubin") else
                         ["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
    m = {}
    cur_fn = None
    line = None
    for ln in out.split("\n"):
        if ln.startswith(".text.") or ln.startswith("\t.section\t.text."):
            cur_fn = ln.split(".text.")[1].split(",")[0].rstrip(":")
        g = re.search(r'File "([^"]+)", line (\d+)', ln)
        if "## File" in ln and g:
            line = (g.group(1).split("/")[-1], int(g.group(2)))
        a = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if a and cur_fn == func:
            m[int(a.group(1), 16)] = line
    return m


def main():
    rep, binary, func = sys.argv[1:4]
    srcdir = sys.argv[4] if len(sys.argv) > 4 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    data = rows[2:]
    ia, iall = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(data[0][ia], 16)
    lines = sass_lines(binary, func)
    agg = Counter()
    for r in data:
        off = int(r[ia], 16) - base
        agg[lines.get(off)] += int(r[iall])
    tot = sum(agg.values())
    cache = {}
    for key, v in agg.most_common(45):
        s = ""
        if srcdir and key:
            fn, ln = key
            if fn not in cache:
                try:
                    cache[fn] = open(f"{srcdir}/{fn}").read().split("\n")
                except OSError:
                    cache[fn] = []
            s = cache[fn][ln - 1].strip()[:80] if ln <= len(cache[fn]) else ""
        print(f"{v:7d} {100 * v / tot:5.1f}%  {key}: {s}")


if __name__ == "__main__":
    main()
