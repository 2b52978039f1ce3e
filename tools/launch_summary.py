"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file F):
python tools/launch_summary.py F [regex]"""
import collections, csv, re, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
tot, cnt = collections.OrderedDict(), collections.Counter()
for r in rows:
    if r[-3] != "gpu__time_duration.sum":
        continue
    name = r[4][:80]
    if pat and not pat.search(name):
        continue
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}.get(r[-2], 1e-6)
    tot[name] = tot.get(name, 0.0) + float(r[-1].replace(",", "")) * scale
    cnt[name] += 1
print("| kernel | launches | total ms |\n|---|---|---|")
for k, v in tot.items():
    print(f"| {k} | {cnt[k]} | {v:.3f} |")
