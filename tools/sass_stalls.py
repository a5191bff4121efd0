"""Dev tool: top SASS instructions by one stall reason from an ncu report.
    python tools/sass_stalls.py REP [reason=long_sb] [top=25]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "long_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = rows[1]
col = hdr.index("stall_" + reason)
body = rows[2:]
tot = sum(int(r[4]) for r in body if r[4].isdigit())
vals = [(int(r[col]), i, r[1].strip()) for i, r in enumerate(body) if r[col].isdigit()]
print(f"total samples {tot}; {reason} {sum(v for v, _, _ in vals)}")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(int(r[hdr.index(h)]) for r in body if r[hdr.index(h)].isdigit()) for h in reasons}
print({k[6:]: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v})
for v, i, src in sorted(vals, reverse=True)[:top]:
    print(f"{v:6d} {i:6d} {src[:90]}")
