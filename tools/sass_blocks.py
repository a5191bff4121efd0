"""Dev tool: basic-block sizes of one kernel's SASS (cuobjdump -sass output)."""
import re, sys
lines = open(sys.argv[1]).read().splitlines()
ins = []
for l in lines:
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
starts = {ins[0][0]}
for i, (a, t) in enumerate(ins):
    m = re.search(r'\bBRA\b.*?(0x[0-9a-f]+)', t)
    if m or 'BAR.SYNC' in t or 'EXIT' in t or 'RET' in t or 'CALL' in t:
        if m: starts.add(int(m.group(1), 16))
        if i + 1 < len(ins): starts.add(ins[i + 1][0])
blocks = []; cur = None
for a, t in ins:
    if a in starts:
        cur = [a, []]; blocks.append(cur)
    cur[1].append(t)
print(f"{len(ins)} instructions, {len(blocks)} blocks, {sum('BAR.SYNC' in t for _, t in ins)} BAR.SYNC")
top = sorted(blocks, key=lambda b: -len(b[1]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for a, ts in top:
    op = lambda p: sum(1 for t in ts if re.search(p, t))
    print(f"@{a:#07x} n={len(ts):5d} LDS={op(r'LDS')} STS={op(r'STS')} FFMA={op(r'FFMA')} FMUL={op(r'FMUL')} FADD={op(r'FADD')} LDG={op(r'LDG')} MUFU={op(r'MUFU')} IMAD/IADD={op(r'IMAD|IADD|LEA')}")
