"""Summarise an ncu report: key throughput metrics, stall reasons and the
hottest SASS lines.  python tools/ncu_summary.py <report.ncu-rep> [--sass N]"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum',
        'smsp__inst_executed_op_shared_atom.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size']


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index('--sass') + 1]) if '--sass' in sys.argv else 0
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(hdr, row))
        print('==', d.get('Kernel Name', '')[:90])
        for k in KEYS:
            if k in d:
                print(f"  {k:64s} {d[k]} {units[hdr.index(k)]}")
        keys = [k for k in hdr if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued')]
        vals = sorted(((float(d[k].replace(',', '')) if d[k] not in ('', 'n/a') else 0, k) for k in keys), reverse=True)
        tot = sum(v for v, _ in vals) or 1
        print('  stalls: ' + ', '.join(f"{k.split('stalled_')[1]} {v / tot * 100:.1f}%" for v, k in vals[:7]))
    if nsass:
        src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(src)))
        hdr = rows[1]
        ix = {h: i for i, h in enumerate(hdr)}
        data = [x for x in rows[2:] if len(x) == len(hdr)]
        tot = sum(int(x[ix['Warp Stall Sampling (All Samples)']]) for x in data) or 1
        top = sorted(data, key=lambda x: -int(x[ix['Warp Stall Sampling (All Samples)']]))[:nsass]
        for x in top:
            print(f"  {int(x[ix['Warp Stall Sampling (All Samples)']]) / tot * 100:5.1f}% "
                  f"{int(x[ix['Instructions Executed']]):10d} {x[ix['Source']][:90]}")


if __name__ == '__main__':
    main()


def opcode_mix(rep, min_exec=100000):
    """Executed warp-instructions per opcode (hot code only)."""
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    mix = {}
    for x in rows[2:]:
        if len(x) != len(hdr):
            continue
        n = int(x[ix['Instructions Executed']])
        if n < min_exec:
            continue
        op = x[ix['Source']].split()
        op = [t for t in op if not t.startswith('@')]
        key = op[0].split('.')[0] if op else '?'
        mix[key] = mix.get(key, 0) + n
    tot = sum(mix.values())
    for k, v in sorted(mix.items(), key=lambda kv: -kv[1]):
        print(f"  {k:12s} {v:12d} {v / tot * 100:5.1f}%")
