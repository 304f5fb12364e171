"""Summarise an ncu --csv launch list: per-kernel total time, share, count, SIMT efficiency."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]
ki, mi, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
idi = h.index('ID')
per = collections.defaultdict(dict)
names = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi: continue
    per[r[idi]][r[mi]] = float(r[vi].replace(',', ''))
    names[r[idi]] = r[ki].split('(')[0][:40]
tot = collections.defaultdict(float); cnt = collections.Counter(); simt = collections.defaultdict(float)
for i, m in per.items():
    t = m.get('gpu__time_duration.sum', 0.0)
    n = names[i]
    tot[n] += t; cnt[n] += 1
    simt[n] += t * m.get('smsp__thread_inst_executed_per_inst_executed.ratio', 0.0)
S = sum(tot.values())
print(f"total {S/1e6:.3f} ms over {sum(cnt.values())} launches")
for n, t in sorted(tot.items(), key=lambda x: -x[1])[:15]:
    print(f"{t/1e6:10.3f} ms {100*t/S:5.1f}%  n={cnt[n]:5d}  simt={simt[n]/max(t,1):5.1f}  {n}")
