#!/usr/bin/env python3
"""Summarise ncu captures from gpurun_out/ into profiles/ (round-tagged markdown + JSON).

  python scripts/summarize_ncu.py --round 1 --launches gpurun_out/launches.csv \
      --rep gpurun_out/prof_b2.ncu-rep --rep gpurun_out/prof_tc.ncu-rep --bench gpurun_out/bench_full.log
"""
import argparse
import collections
import csv
import json
import os
import subprocess

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed']


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == 'ID':
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d['Metric Name'] != 'gpu__time_duration.sum':
            continue
        name = d['Kernel Name'].split('(')[0]
        v = float(d['Metric Value'].replace(',', ''))
        scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}.get(d['Metric Unit'], 1e-3)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k[:80]}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% |")
    return "\n".join(out)


def rep_kernels(path):
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, u = rr[0], rr[1]
    res = []
    for v in rr[2:]:
        k = {key: (v[h.index(key)], u[h.index(key)]) for key in KEYS if key in h}
        st = [(x, float(v[i])) for i, x in enumerate(h)
              if x.startswith('smsp__average_warps_issue_stalled') and x.endswith('per_issue_active.ratio')]
        st = sorted(st, key=lambda t: -t[1])[:6]
        name = v[h.index('Kernel Name')] if 'Kernel Name' in h else '?'
        res.append((name, k, st))
    return res


def to_bytes(val, unit):
    return float(val) * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument('--round', type=int, default=1)
    ap.add_argument('--launches')
    ap.add_argument('--rep', action='append', default=[])
    ap.add_argument('--bench')
    ap.add_argument('--dominant', default='b2search')
    a = ap.parse_args()
    os.makedirs('profiles', exist_ok=True)
    md = [f"# Round {a.round} profiles (B200, ncu --clock-control none)\n"]
    if a.bench:
        b = json.loads(open(a.bench).read().strip().splitlines()[-1])
        md.append(f"Bench line (`python bench.py`, C3): {b['ms_per_step']:.3f} ms per 512x512 encode, "
                  f"{b['value']:.3e} pairs/s; e2e {b.get('e2e', {}).get('value', 0):.3e} pairs/s; "
                  f"roofline frac {b['roofline']['frac']:.3f} ({b['roofline']['kernel']}).\n")
        md.append("| B | ranges | kept | pairs | exact evals | pool ms | search ms |\n|---|---|---|---|---|---|---|")
        for l in b['levels']:
            md.append(f"| {l['B']} | {l['n_ranges']} | {l['n_kept']} | {l['pairs']:.3e} | {l['exact_evals']} | "
                      f"{l['ms_pool']:.3f} | {l['ms_search']:.3f} |")
        md.append("")
    if a.launches:
        md.append("## Launch list (`bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e`: 3 warm-up, 2 timed and 2 instrumented encodes; cold-cache serialised: compare shares)\n")
        md.append(launch_table(a.launches))
        md.append("")
    summary = {"round": a.round, "kernels": []}
    for rep in a.rep:
        for name, k, st in rep_kernels(rep):
            md.append(f"## `{name}`\n")
            md.append("| metric | value |\n|---|---|")
            for key, (val, unit) in k.items():
                md.append(f"| {key} | {val} {unit} |")
            md.append("\nTop stalls (warps per issue-active cycle): " +
                      ", ".join(f"{x.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {y:.2f}" for x, y in st) + "\n")
            ent = {"kernel": name, "metrics": {key: {"value": val, "unit": unit} for key, (val, unit) in k.items()}}
            if 'dram__bytes_read.sum' in k and 'dram__bytes_write.sum' in k:
                ent["dram_bytes"] = to_bytes(*k['dram__bytes_read.sum']) + to_bytes(*k['dram__bytes_write.sum'])
            summary["kernels"].append(ent)
            if a.dominant in name and "search_dram_bytes_per_launch" not in summary:
                summary["search_dram_bytes_per_launch"] = ent.get("dram_bytes")
                summary["dominant_kernel"] = name
    open(f"profiles/r{a.round:02d}_summary.md", "w").write("\n".join(md) + "\n")
    json.dump(summary, open("profiles/ncu_summary.json", "w"), indent=1)
    print("\n".join(md))


if __name__ == '__main__':
    main()
