"""Dev tool: per-source-line warp-stall samples from an ncu report
(ncu -i REP --page source --csv --print-source cuda,sass)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
f = None; hdr = None; rows = []; tot = 0
for rec in csv.reader(out):
    if not rec: continue
    if rec[0] == "File Path": f = rec[1].split("/")[-1]; continue
    if rec[0] == "Line No": hdr = rec; continue
    if rec[0] in ("Function Name",) or hdr is None: continue
    if rec[0] and rec[0] != "":
        try: s = int(rec[4]); ins = int(rec[7])
        except ValueError: continue
        rows.append((s, ins, f, rec[0], rec[1].strip()[:90])); tot += s
rows.sort(reverse=True)
print(f"total samples {tot}")
byfile = collections.Counter()
for s, ins, f, ln, src in rows: byfile[f] += s
print(dict(byfile))
for s, ins, f, ln, src in rows[:top]:
    print(f"{100*s/tot:5.1f}% {ins:>10d} {f}:{ln}  {src}")
