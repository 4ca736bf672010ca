# summarise an ncu launch-list csv: count, avg us, name
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv')) if len(r) > 5]
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
c = collections.Counter(); t = collections.defaultdict(float)
for r in rows[1:]:
    n = r[ki][:60]; c[n] += 1; t[n] += float(r[vi].replace(',', ''))
for n in c:
    print(c[n], round(t[n] / c[n] / 1e3, 1), n)
