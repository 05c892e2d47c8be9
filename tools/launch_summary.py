"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count / median / total.
usage: launch_summary.py <csv> [first_n_launches]"""
import csv, collections, sys
lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
limit = int(sys.argv[2]) if len(sys.argv) > 2 else None
for r in rows[1:limit + 1 if limit else None]:
    if len(r) > iv:
        d[r[ik].split("(")[0][:48]].append(float(r[iv].replace(",", "")) / 1000)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:50s} n={len(v):5d} median={sorted(v)[len(v)//2]:9.2f} us  total={sum(v):10.1f} us  share={sum(v)/tot:.3f}")
