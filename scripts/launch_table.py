#!/usr/bin/env python3
"""Aggregate an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == 'ID':
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d['Metric Name'] != 'gpu__time_duration.sum':
                continue
            v = float(d['Metric Value'].replace(',', ''))
            u = d['Metric Unit']
            us = v / 1000 if u == 'nsecond' else v * 1000 if u == 'msecond' else v
            n = d['Kernel Name'].split('(')[0][:80]
            agg[n][0] += 1
            agg[n][1] += us
    tot = sum(v[1] for v in agg.values()) or 1
    print('| kernel | launches | total us | share |\n|---|---|---|---|')
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f'| `{n}` | {c} | {t:.1f} | {100 * t / tot:.1f}% |')
    print(f'| total | | {tot:.1f} | |')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
