import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            out.append((d['Kernel Name'].split('(')[0], float(d['Metric Value']) * (1e-3 if d['Metric Unit'] == 'ns' else 1)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(out)
tail = out[-n:]
tot = sum(t for _, t in tail)
for k, t in tail: print(f"{k:50s} {t:9.2f} us  {100*t/tot:5.1f}%")
print("total", round(tot, 2), "us")
