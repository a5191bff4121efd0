"""Dev tool: unique hazard sites of a compute-sanitizer racecheck log.

    python tools/racecheck_summary.py gpurun_out/sanitize/racecheck.log
"""
import collections
import re
import sys

pat = re.compile(r"\((.+?)\) Potential (\w+) hazard detected at __shared__ \S+ in block")
acc = re.compile(r"(Read|Write) Thread \((\d+),\d+,\d+\) at (.+?) in (\S+)")
cnt = collections.Counter()
cur = None
for line in open(sys.argv[1], errors="replace"):
    m = pat.search(line)
    if m:
        cur = [m.group(1), m.group(2)]
        continue
    m = acc.search(line)
    if m and cur is not None:
        cur.append(f"{m.group(1)} t{m.group(2)} {m.group(3)} {m.group(4)}")
        if len(cur) == 4:
            key = (cur[0], cur[1], re.sub(r" t\d+", "", cur[2]), re.sub(r" t\d+", "", cur[3]))
            cnt[key] += 1
            cur = None
for k, v in cnt.most_common():
    print(v, *k, sep="\n   ")
tail = [l for l in open(sys.argv[1], errors="replace") if "SUMMARY" in l or " rc=" in l]
print("".join(tail))
