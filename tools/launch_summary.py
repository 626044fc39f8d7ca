"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel (name, grid) launches, total us, average us, share."""
import csv, collections, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    gi = h.index('Grid Size') if 'Grid Size' in h else None
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi or not r[vi].replace(',', '').replace('.', '').isdigit():
            continue
        out.append((r[ki].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', ''),
                    r[gi] if gi is not None else '', float(r[vi].replace(',', '')) / 1000.0))
    return out

if __name__ == '__main__':
    data = load(sys.argv[1])
    lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    hi = int(sys.argv[3]) if len(sys.argv) > 3 else len(data)
    data = data[lo:hi]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, g, us in data:
        a = agg[(k, g)]; a[0] += 1; a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"{len(data)} launches, {tot:.1f} us")
    print("| kernel | grid | launches | total us | avg us | share |\n|---|---|---|---|---|---|")
    for (k, g), (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {g} | {n} | {us:.1f} | {us/n:.2f} | {us/tot:.3f} |")
