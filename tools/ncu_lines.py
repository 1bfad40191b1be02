"""Aggregate ncu 'cuda,sass' source-page stall samples by CUDA source line -- dev tool.
usage: ncu -i rep --page source --csv --print-source cuda,sass > f.csv; ncu_lines.py f.csv [n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'Line No')
h = rows[hi]
st = [i for i, x in enumerate(h) if x.startswith('stall_') and 'Not Issued' not in x]
agg = collections.Counter()
det = collections.defaultdict(collections.Counter)
src = {}
cur = None
tot = 0
fname = ''
for r in rows[hi + 1:]:
    if len(r) < 5:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0]:
        if not r[0].isdigit():
            continue
        cur = (fname, int(r[0]))
        src[cur] = r[1]
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    agg[cur] += s
    tot += s
    for i in st:
        try:
            det[cur][h[i]] += float(r[i] or 0)
        except ValueError:
            pass
print("total samples", tot)
for ln, s in agg.most_common(n):
    top = ", ".join(f"{k[6:]}={int(v)}" for k, v in det[ln].most_common(3))
    print(f"{ln[0][:10]}:{ln[1]:5d} {100 * s / tot:5.1f}%  {src.get(ln, '').strip()[:64]:64s} {top}")
