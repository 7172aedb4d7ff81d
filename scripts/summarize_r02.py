#!/usr/bin/env python3
"""Round-2 profile summary: profiles/r02_summary.md + profiles/ncu_summary.json from the CSV
exports of the round-2 ncu captures (scripts/refresh_profiles_r02.sh), the launch list and the
bench lines.  HBM fractions use MEASURED_PEAKS.json hbm_gbs (6552 GB/s)."""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_ncu import launch_table  # noqa: E402

MUL = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-9, 'usecond': 1e-6, 'msecond': 1e-3,
       'ns': 1e-9, 'us': 1e-6, 'ms': 1e-3}


def load(path):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    return [(dict(zip(h, v)), dict(zip(h, u))) for v in rows[2:]]


def val(d, u, k):
    x = d.get(k)
    if not x:
        return None
    return float(x.replace(',', '')) * MUL.get(u.get(k, ''), 1)


def main():
    hbm = json.load(open('MEASURED_PEAKS.json')).get('hbm_gbs', 6552.0) if os.path.exists('MEASURED_PEAKS.json') else 6552.0
    md = ['# Round 2 profiles (B200, ncu --clock-control none, --set full; cold-cache serialised launches)\n']
    for name, path in (('C3 (headline)', 'gpurun_out/bench_r02.log'), ('C4', 'gpurun_out/bench_c4_r02.log'),
                       ('C5', 'gpurun_out/bench_c5_r02.log')):
        if not os.path.exists(path):
            continue
        b = json.loads(open(path).read().strip().splitlines()[-1])
        md.append(f"**{name}** (`{' '.join(['bench.py'] + (['--config', b['config']['workload']] if b['config']['workload'] != 'C3' else []))}`): "
                  f"{b['ms_per_step']:.3f} ms per encode, {b['value']:.3e} effective pairs/s, "
                  f"{b['evaluated_pairs_per_s']:.3e} evaluated pairs/s, roofline frac {b['roofline']['frac']:.3f} "
                  f"({b['roofline']['kernel']}), clocks {b['clocks'].get('sm_mhz')} MHz {b['clocks'].get('reasons')}"
                  + (f", parity {b['parity']}" if 'parity' in b else '') + "\n")
        md.append('| B | ranges | kept | pairs | evaluated | exact | search ms | roof frac |\n|---|---|---|---|---|---|---|---|')
        for l in b['levels']:
            md.append(f"| {l['B']} | {l['n_ranges']} | {l['n_kept']} | {l['pairs']:.3e} | {l['pairs_scanned'] * 8:.3e} | "
                      f"{l['exact_evals']} | {l['ms_search']:.3f} | {l['roof_frac']:.3f} |")
        md.append('')
    if os.path.exists('gpurun_out/launches_r02.csv'):
        md.append('## Launch list of the C3 bench (`bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e`)\n')
        md.append(launch_table('gpurun_out/launches_r02.csv'))
        md.append('')
    summary = {'round': 2, 'hbm_gbs_peak': hbm, 'kernels': []}
    for title, path in (('every kernel of one C3 encode', 'gpurun_out/prof_c3_r02_raw.csv'),
                        ('pool kernels of one C5 encode (4096^2)', 'gpurun_out/prof_c5pool_r02_raw.csv')):
        if not os.path.exists(path):
            continue
        md.append(f'## {title}: DRAM traffic and HBM fraction\n')
        md.append('| kernel | us | DRAM MB (r+w) | GB/s | of HBM peak | L2 % | issue active % |\n|---|---|---|---|---|---|---|')
        for d, u in load(path):
            n = d['Kernel Name'].split('(')[0].replace('fic::', '')
            t = val(d, u, 'gpu__time_duration.sum')
            by = (val(d, u, 'dram__bytes_read.sum') or 0) + (val(d, u, 'dram__bytes_write.sum') or 0)
            gbs = by / t / 1e9
            md.append(f"| `{n[:60]}` | {t * 1e6:.1f} | {by / 1e6:.2f} | {gbs:.1f} | {gbs / hbm:.3f} | "
                      f"{float(d.get('lts__throughput.avg.pct_of_peak_sustained_elapsed') or 0):.1f} | "
                      f"{float(d.get('smsp__issue_active.avg.pct_of_peak_sustained_active') or 0):.1f} |")
            summary['kernels'].append({'kernel': d['Kernel Name'], 'capture': title, 'us': t * 1e6, 'dram_bytes': by,
                                       'gbs': gbs, 'hbm_frac': gbs / hbm})
        md.append('')
    open('profiles/r02_summary.md', 'w').write('\n'.join(md) + '\n')
    json.dump(summary, open('profiles/ncu_summary.json', 'w'), indent=1)
    print('\n'.join(md))


if __name__ == '__main__':
    main()
