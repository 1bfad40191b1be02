"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if 'Kernel Name' in r:
        hdr = r; start = i + 1; break
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[start:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].split('<')[0]
    us = float(r[vi].replace(',', '')) * scale[r[ui]]
    tot[name] += us; cnt[name] += 1
S = sum(tot.values())
print(f"launches {sum(cnt.values())}, total device time {S:.1f} us")
for k, v in tot.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 15):
    print(f"  {k:28s} n={cnt[k]:6d} total={v:11.1f}us ({100*v/S:5.1f}%) avg={v/cnt[k]:8.2f}us")
