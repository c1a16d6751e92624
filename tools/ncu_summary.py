"""Summarise an ncu --set full capture (raw CSV + SASS source CSV) for profiles/."""
import collections
import csv
import re
import sys


def num(x):
    try:
        return float(str(x).replace(',', ''))
    except ValueError:
        return None


def raw_summary(path):
    r = list(csv.reader(open(path)))
    d = dict(zip(r[0], r[2]))
    keys = ['gpu__time_duration.sum', 'sm__cycles_elapsed.avg', 'smsp__inst_executed.sum',
            'sm__inst_executed.avg.per_cycle_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
            'sm__warps_active.avg.per_cycle_active',
            'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed_op_shared_atom.sum',
            'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum',
            'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
            'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
            'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
            'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
            'l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed',
            'lts__t_sectors.sum', 'launch__registers_per_thread']
    out = {}
    for k in keys:
        if k in d:
            out[k] = d[k]
    stalls = {k.replace('smsp__pcsamp_warps_issue_stalled_', ''): num(v) for k, v in d.items()
              if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued')}
    return out, stalls


def sass_summary(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    byop, samp = collections.Counter(), collections.Counter()
    for d in data:
        m = re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_]+(\.[A-Z0-9_]+)*)', d['Source'].strip())
        if not m:
            continue
        byop[m.group(2)] += num(d['Instructions Executed']) or 0
        samp[m.group(2)] += num(d['Warp Stall Sampling (All Samples)']) or 0
    return byop, samp


if __name__ == '__main__':
    raw, stalls = raw_summary(sys.argv[1])
    for k, v in raw.items():
        print(f"{k:70s} {v}")
    tot = sum(v for v in stalls.values() if v)
    print("\nstall samples (share):")
    for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0))[:12]:
        print(f"  {k:30s} {100 * (v or 0) / tot:6.2f}%")
    if len(sys.argv) > 2:
        byop, samp = sass_summary(sys.argv[2])
        ti, ts = sum(byop.values()), sum(samp.values())
        print("\ninstruction mix (executed share / stall-sample share):")
        for op, c in byop.most_common(25):
            print(f"  {op:28s} {100 * c / ti:6.2f}%  {100 * samp[op] / ts:6.2f}%")
