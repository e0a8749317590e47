"""Static SASS look at a join kernel's hot loop: finds the unmasked rotation (the FFMA/FFMA2
region with no FSEL -INF masking) and prints its opcode histogram per cell.
usage: python tools/sass_loop.py <lib.so> <function-substring> <cells-per-iteration>"""
import collections, re, subprocess, sys
lib, pat, cells = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
body = [f for f in funcs if f.split("\n", 1)[0].strip().find(pat) >= 0]
assert body, "function not found"
ins = []
for l in body[0].splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
# loops: backward branches
loops = []
for k, (a, x) in enumerate(ins):
    m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)\s*$", x) if "BRA" in x else None
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a:
            seg = [y for b, y in ins if tgt <= b <= a]
            loops.append((tgt, a, seg))
def op(x):
    x = re.sub(r"^@!?U?P\w+\s+", "", x)
    return x.split()[0]
best = None
for tgt, a, seg in loops:
    c = collections.Counter(op(x).split(".")[0] for x in seg)
    fp = c["FFMA"] + c["FFMA2"]
    masked = sum(1 for x in seg if "-INF" in x)
    if fp and masked == 0 and (best is None or fp > best[3] or (fp == best[3] and len(seg) < len(best[2]))):
        best = (tgt, a, seg, fp)
for tgt, a, seg in loops:
    c = collections.Counter(op(x).split(".")[0] for x in seg)
    print(f"loop {tgt:#x}-{a:#x}: {len(seg)} instr, FFMA {c['FFMA']} FFMA2 {c['FFMA2']} -INF {sum(1 for x in seg if '-INF' in x)}")
if best:
    tgt, a, seg, _ = best
    c = collections.Counter(op(x) for x in seg)
    print(f"\nunmasked hot loop {tgt:#x}-{a:#x}: {len(seg)} instructions = {len(seg)/cells:.2f} per cell")
    for k, v in c.most_common(40):
        print(f"  {k:28s} {v:4d}  {v/cells:.3f}/cell")
