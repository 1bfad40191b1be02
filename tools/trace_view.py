"""Summaries of a kernel timeline written by trace_hlu.py (dev tool).
usage: trace_view.py trace.json [anchor_index]"""
import collections
import json
import sys

ev = json.load(open(sys.argv[1]))
ev = [e for e in ev if not e['name'].startswith('Mem')]
names = collections.defaultdict(list)
for e in ev:
    names[(e['name'], e['stream'])].append(e['end'] - e['start'])
for (n, s), v in sorted(names.items(), key=lambda x: -sum(x[1])):
    print(f"{n:16s} stream {s:3d} {len(v):5d} mean {sum(v)/len(v):7.1f} us  tot {sum(v)/1e3:7.2f} ms")
t0 = ev[0]['start']
print("span ms", (max(e['end'] for e in ev) - t0) / 1e3)
lus = [e for e in ev if e['name'].startswith('k_h2_lu')]
ai = int(sys.argv[2]) if len(sys.argv) > 2 else 30
a, b = lus[ai]['start'], lus[ai + 2]['start']
for e in ev:
    if a - 50 <= e['start'] <= b:
        print(f"{e['stream']:3d} {e['name']:16s} {e['start']-a:8.1f} {e['end']-a:8.1f} dur {e['end']-e['start']:6.1f}")
