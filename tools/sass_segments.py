"""Segments an `ncu --page source --csv` dump into runs of SASS with equal execution counts:
share of executed instructions and of stall samples per run (where a kernel's time goes)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if 'Instructions Executed' in r)
ia = hdr.index('Instructions Executed'); isamp = hdr.index('# Samples'); isrc = hdr.index('Source')
body = [r for r in rows if len(r) > max(ia, isamp) and r[ia].isdigit()]
tot = sum(int(r[ia]) for r in body); ts = sum(int(r[isamp]) for r in body)
print('total instr', tot, 'samples', ts, 'n sass', len(body))
seg = []
for i, r in enumerate(body):
    n = int(r[ia]); s = int(r[isamp])
    if seg and abs(seg[-1][2] - n) <= 0.05 * max(n, 1):
        seg[-1][1] = i; seg[-1][3] += n; seg[-1][4] += s
    else:
        seg.append([i, i, n, n, s])
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for a, b, n, sumn, s in seg:
    if sumn > thr * tot or s > thr * ts:
        print(f"sass {a:4d}-{b:4d} exec/instr {n:8d} instrs {100*sumn/tot:5.1f}% samples {100*s/ts:5.1f}%  first: {body[a][isrc].strip()[:70]}")
