"""Per VOTE.ANY-delimited segment of a SASS dump: count FFMA/FMUL/IMAD/FMNMX by number of
non-reused register source operands (3 fresh reads = register-bank conflict candidates)."""
import re, sys, collections
lines = [l for l in open(sys.argv[1]) if re.search(r'/\*[0-9a-f]{4}\*/', l)]
segs, cur = [], []
for l in lines:
    cur.append(l)
    if 'VOTE.ANY' in l:
        segs.append(cur); cur = []
for k, seg in enumerate(segs):
    cnt = collections.Counter()
    for line in seg:
        m = re.search(r'\s(FFMA|FMUL|IMAD|FMNMX3|FMNMX)\s+(.*?);', line)
        if not m:
            continue
        ops = [o.strip() for o in m.group(2).split(',')][1:]
        fresh = 0
        for o in ops:
            r = re.match(r'-?\|?(R\d+)(\.reuse)?', o)
            if r and r.group(1) != 'RZ' and not r.group(2):
                fresh += 1
        cnt[(m.group(1), fresh)] += 1
    n3 = sum(v for (op, f), v in cnt.items() if f >= 3)
    nffma = sum(v for (op, f), v in cnt.items() if op == 'FFMA')
    print(f"seg {k}: instr {len(seg)} FFMA {nffma} three-fresh {n3}  " +
          " ".join(f"{op}{f}:{v}" for (op, f), v in sorted(cnt.items())))
