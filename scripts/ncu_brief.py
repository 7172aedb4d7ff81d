#!/usr/bin/env python3
"""Print the key metrics, stall reasons and the hottest source lines of every kernel in an
ncu report (read locally: ncu -i REP --page raw/source --csv)."""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'smsp__inst_executed.sum',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum']


def main(rep, nlines=25):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print('==', d.get('Kernel Name', '')[:90])
        for k in KEYS:
            print('  %-72s %s' % (k, d.get(k)))
        st = []
        for k, v in d.items():
            if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
                try:
                    st.append((float(v), k.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print('  stalls:', ', '.join('%s %.0f%%' % (k, 100 * v / tot) for v, k in sorted(st, reverse=True)[:8]))
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    blocks = src.split('"File Path"')
    for blk in blocks[1:]:
        rows = list(csv.reader(io.StringIO('"File Path"' + blk)))
        fn = rows[1][1] if len(rows) > 1 else ''
        hdr = rows[2]
        iL, iI, iT, iW = (hdr.index(x) for x in ('Line No', 'Instructions Executed', 'Thread Instructions Executed',
                                                  'Warp Stall Sampling (All Samples)'))
        out = []
        for r in rows[3:]:
            if len(r) < len(hdr) or not r[iL]:
                continue
            try:
                out.append((float(r[iI]), float(r[iT]), float(r[iW]), r[iL], r[1][:100]))
            except ValueError:
                pass
        ti = sum(o[0] for o in out) or 1
        tw = sum(o[2] for o in out) or 1
        print('== source:', fn[:90], 'inst %.3g' % ti)
        for o in sorted(out, key=lambda x: -x[2])[:nlines]:
            print('  %5.1f%% inst %5.1f%% stall thr/inst %4.1f L%s: %s' % (100 * o[0] / ti, 100 * o[2] / tw,
                                                                           o[1] / max(o[0], 1), o[3], o[4]))


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
