"""Per-source-line stall summary of an ncu --set full report.

usage: python tools/ncu_hot.py <report.ncu-rep> [top] [--sass]
Reads `ncu -i <rep> --page source --csv --print-source cuda,sass` (needs a
-lineinfo build and --import-source on), keeps the CUDA-line rows (which carry
the metrics aggregated over their SASS), and prints the lines with the most
warp-stall samples and their top stall reasons.  --sass lists instructions.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25
want_sass = "--sass" in sys.argv
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], "", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    rows.append((fname, r))
h = hdr
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


sel = [(fn, r) for fn, r in rows if (r[0] == "") == want_sass]
tot = sum(f(r[si]) for _, r in sel)
print(f"total stall samples {tot:.0f}")
for fn, r in sorted(sel, key=lambda x: -f(x[1][si]))[:top]:
    s = f(r[si])
    reasons = sorted(((f(r[i]), h[i][6:]) for i in stall_cols), reverse=True)[:3]
    rs = " ".join(f"{n}:{100 * v / max(s, 1):.0f}%" for v, n in reasons if v > 0)
    text = (r[3] if want_sass else r[1]).strip()[:80]
    loc = r[2] if want_sass else f"{fn}:{r[0]}"
    print(f"{100 * s / max(tot, 1):5.1f}% {loc:>22} inst={int(f(r[ie])):>10} | {text} | {rs}")
