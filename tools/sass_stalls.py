"""Top SASS lines per stall reason from an ncu source-page CSV (ncu -i X --page source --csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
isrc = h.index("Source")
reasons = sys.argv[2].split(",") if len(sys.argv) > 2 else ["stall_long_sb", "stall_wait", "stall_short_sb"]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
for rsn in reasons:
    col = h.index(rsn)
    lst = sorted(((int(r[col] or 0), i, r[isrc].strip()) for i, r in enumerate(data)), reverse=True)
    tot = sum(x[0] for x in lst)
    print(f"== {rsn}: {tot}")
    for s, i, src in lst[:n]:
        print(f"{s:6d} {i:5d} {src}")
