"""Summarise an ncu --set full capture (raw + sass CSV exports): key counters, stall mix, top stalled SASS."""
import csv
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'lts__t_sector_hit_rate.pct', 'smsp__warps_active.avg.per_cycle_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'smsp__inst_executed.sum', 'launch__registers_per_thread', 'launch__block_size', 'launch__grid_size']


def main(raw, sass=None, top=25):
    top = int(top)
    r = list(csv.reader(open(raw)))
    hdr = r[0]
    st = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued')]
    for row in r[2:]:
        print(row[hdr.index('Kernel Name')][:90])
        for k in KEYS:
            if k in hdr:
                print('  ', k, row[hdr.index(k)])
        tot = sum(float(row[hdr.index(h)].replace(',', '')) for h in st)
        for h in sorted(st, key=lambda h: -float(row[hdr.index(h)].replace(',', '')))[:8]:
            print('    stall', h.replace('smsp__pcsamp_warps_issue_stalled_', ''),
                  round(float(row[hdr.index(h)].replace(',', '')) / tot * 100, 1))
    if not sass:
        return
    rows = list(csv.reader(open(sass)))
    hi = [i for i, x in enumerate(rows) if x and x[0] == 'Address'][0]
    hdr = rows[hi]
    data = []
    for x in rows[hi + 1:]:
        if x and x[0] == 'Address':
            break
        if len(x) == len(hdr) and x[0].startswith('0x'):
            data.append(x)
    iS = hdr.index('Warp Stall Sampling (All Samples)')
    iE = hdr.index('Instructions Executed')
    tot = sum(int(x[iS]) for x in data)
    print('samples', tot)
    for x in sorted(data, key=lambda x: -int(x[iS]))[:top]:
        print(x[0][-5:], x[iS].rjust(7), round(int(x[iS]) / tot * 100, 1), x[iE].rjust(9), x[1][:80])


if __name__ == '__main__':
    main(*sys.argv[1:])
