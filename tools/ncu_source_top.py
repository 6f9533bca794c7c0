"""Top source / SASS lines of an ncu report by a metric column (read with `ncu -i --page source`).

usage: python tools/ncu_source_top.py <report.ncu-rep> [substring-of-column ...] [--n 25] [--sass]
Columns are matched by substring (case-insensitive), e.g. "bank conflicts", "stall sampling".
"""
import csv
import io
import subprocess
import sys


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n = 25
    if "--n" in sys.argv:
        n = int(sys.argv[sys.argv.index("--n") + 1])
        args = [a for a in args if a != str(n)]
    view = "sass" if "--sass" in sys.argv else "cuda"
    path, wanted = args[0], [w.lower() for w in args[1:]] or ["stall sampling (all samples)"]
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    if "--dump" in sys.argv:
        print(raw[:3000])
    rows = list(csv.reader(io.StringIO(raw)))
    hdr_i = next(i for i, r in enumerate(rows) if any("Warp Stall Sampling" in h for h in r))
    hdr = rows[hdr_i]
    print("columns:", " | ".join(hdr))
    src_col = next((i for i, h in enumerate(hdr) if h.lower() in ("source", "sass", "address")), 1)
    for w in wanted:
        cols = [i for i, h in enumerate(hdr) if w in h.lower()]
        if not cols:
            print(f"no column matching {w!r}")
            continue
        c = cols[0]

        def val(r):
            try:
                return float(r[c].replace(",", ""))
            except (ValueError, IndexError):
                return 0.0

        body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r != hdr]
        tot = sum(val(r) for r in body) or 1.0
        print(f"\n== top {n} by {hdr[c]} (total {tot:.0f})")
        for r in sorted(body, key=val, reverse=True)[:n]:
            extra = {h: r[i] for i, h in enumerate(hdr) if h in ("Instructions Executed", "L1 Wavefronts Shared",
                                                                  "L1 Wavefronts Shared Ideal")}
            print(f"{val(r):12.0f} {100 * val(r) / tot:5.1f}%  " + " | ".join(x[:90] for x in r[:2]) + f"  {extra}")


if __name__ == "__main__":
    main()
