"""Dynamic instruction mix of an ncu report: warp instructions executed per SASS opcode.

usage: python tools/ncu_opcode_mix.py <report.ncu-rep> [--n 30]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 30
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    hdr = rows[hi]
    si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
    mix = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) != len(hdr) or r == hdr:
            continue
        txt = r[si].strip()
        if txt.startswith("@"):
            txt = txt.split(None, 1)[1] if " " in txt else txt
        op = txt.split()[0] if txt else "?"
        try:
            mix[op] += int(float(r[ei].replace(",", "")))
        except ValueError:
            pass
    tot = sum(mix.values()) or 1
    print(f"total warp instructions {tot}")
    for op, c in mix.most_common(n):
        print(f"{op:28s} {c:14d} {100 * c / tot:6.2f}%")


if __name__ == "__main__":
    main()
