"""Summarises an ncu launch list (gpu__time_duration per launch, cold-cache, serialised): the
kernels of one steady assemble step (the launches between the last two tile-kernel groups) and
each kernel's share of that step."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
seq = [(r[ix['Kernel Name']].split('(')[0].replace('void ', ''), float(r[ix['Metric Value']].replace(',', '')))
       for r in rows[1:] if r[ix['Metric Name']] == 'gpu__time_duration.sum']
tile = [i for i, (k, _) in enumerate(seq) if k.startswith('sy_')]
# group tile launches into steps: consecutive sy_ launches separated only by non-sy launches of one step
starts = [tile[0]] + [tile[j] for j in range(1, len(tile)) if any(not seq[m][0].startswith('sy_') for m in range(tile[j - 1] + 1, tile[j]))]
a, b = starts[-2], starts[-1]
step = seq[a:b]
tot = sum(v for _, v in step)
print(f"{len(seq)} launches in the capture; steady step = launches [{a}, {b}) : {len(step)} launches, "
      f"{tot / 1e6:.3f} ms (ncu, serialised, cold caches)")
agg = collections.OrderedDict()
for k, v in step:
    agg.setdefault(k, [0, 0.0]); agg[k][0] += 1; agg[k][1] += v
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {v / tot * 100:5.1f}%  {v / 1e6:8.3f} ms  x{n}  {k[:90]}")
