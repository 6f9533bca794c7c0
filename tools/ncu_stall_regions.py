"""Where a kernel's warps wait: pc-sampling stall samples of an ncu report, per opcode and per
stall reason, plus the hottest SASS instructions with their dominant reasons.

usage: python tools/ncu_stall_regions.py <report.ncu-rep> [--n 50]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 50
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    hdr = rows[hi]
    si = hdr.index("Source")
    samp = next(i for i, h in enumerate(hdr) if h.startswith("Warp Stall Sampling (All"))
    reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]

    def num(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0

    body = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r != hdr]
    total = sum(num(r[samp]) for r in body) or 1.0
    by_op = collections.defaultdict(lambda: collections.Counter())
    for r in body:
        txt = r[si].strip()
        if txt.startswith("@"):
            txt = txt.split(None, 1)[1] if " " in txt else txt
        op = txt.split()[0].split(".")[0] if txt else "?"
        for i, h in reasons:
            by_op[op][h] += num(r[i])
    print(f"total samples {total:.0f}")
    print("== stall samples per opcode (share of all samples; top reasons)")
    tot_op = {op: sum(c.values()) for op, c in by_op.items()}
    for op, t in sorted(tot_op.items(), key=lambda x: -x[1])[:16]:
        top = ", ".join(f"{h.replace('stall_', '')} {100 * v / total:.1f}" for h, v in by_op[op].most_common(4))
        print(f"  {op:10s} {100 * t / total:5.1f}%   {top}")
    print(f"== top {n} instructions")
    for idx, r in sorted(enumerate(body), key=lambda x: -num(x[1][samp]))[:n]:
        c = collections.Counter({h: num(r[i]) for i, h in reasons})
        top = ", ".join(f"{h.replace('stall_', '')} {v:.0f}" for h, v in c.most_common(3) if v)
        print(f"  #{idx:5d} {100 * num(r[samp]) / total:4.1f}%  {r[si].strip()[:70]:70s} {top}")


if __name__ == "__main__":
    main()
