"""Per CUDA source line stall samples from `ncu -i X --page source --csv --print-source cuda,sass`.

  python tools/ncu_lines.py <csv> [n]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        stall = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
    elif hdr and r and r[0] not in ("", "Function Name"):
        try:
            s = float(r[isamp] or 0)
        except ValueError:
            continue
        top = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall), reverse=True)[:2]
        out.append((s, f"{fname}:{r[0]}", r[1].strip()[:90], top))
tot = sum(o[0] for o in out)
for s, loc, src, top in sorted(out, reverse=True)[:n]:
    t = " ".join(f"{k}={100 * v / max(s, 1):.0f}%" for v, k in top)
    print(f"{100 * s / tot:5.1f}% {loc:22s} {t:30s} {src}")
