"""Aggregate an ncu --metrics gpu__time_duration.sum launch list by kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split('(')[0]
        v = float(r[vi].replace(',', ''))
        ms = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0}.get(r[ui], 1e-6) * v
        agg[name][0] += 1
        agg[name][1] += ms
        tot += ms
    print(f"{'kernel':44s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:44s} {n:8d} {ms:10.2f} {100 * ms / tot:6.2f}%")
    print(f"{'total':44s} {sum(v[0] for v in agg.values()):8d} {tot:10.2f}")


if __name__ == '__main__':
    main(sys.argv[1])
