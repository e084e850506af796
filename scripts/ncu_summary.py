"""Summarise an ncu --set full CSV export (scripts/ncu_capture.sh) -> text."""
import csv, gzip, collections, sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Achieved Occupancy', 'Registers Per Thread',
        'Compute (SM) Throughput', 'Grid Size', 'Block Size', 'Theoretical Occupancy', 'L2 Hit Rate',
        'Executed Ipc Active', 'Issue Slots Busy', 'Waves Per SM', 'Block Limit Registers']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum',
       'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
       'smsp__inst_executed.sum', 'launch__grid_size', 'launch__registers_per_thread']


def summary(stem, elems=None):
    out = []
    rows = list(csv.reader(open(stem + '.details.csv')))
    h = rows[0]
    out.append(f"kernel: {dict(zip(h, rows[1])).get('Kernel Name', '?')[:160]}")
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get('Metric Name') in WANT:
            out.append(f"  {d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
    raw = list(csv.reader(open(stem + '.raw.csv')))
    hh = raw[0]
    vals = raw[2] if len(raw) > 2 else raw[1]
    for k in RAW:
        if k in hh:
            out.append(f"  {k}: {vals[hh.index(k)]} {raw[1][hh.index(k)]}")
    try:
        r = list(csv.reader(gzip.open(stem + '.sass.csv.gz', 'rt')))
        h = r[1]
        rows = [dict(zip(h, x)) for x in r[2:] if len(x) == len(h)]
        tot = 0
        ops = collections.Counter()
        for d in rows:
            t = int(d['Thread Instructions Executed'] or 0)
            tot += t
            src = d['Source'].strip().split()
            if not src:
                continue
            op = src[1] if src[0].startswith('@') else src[0]
            ops[op.split('.')[0]] += t
        if elems:
            out.append(f"  thread instructions per element: {tot / elems:.1f}")
            out.append("  top opcodes per element: " + ", ".join(f"{k} {v / elems:.2f}" for k, v in ops.most_common(16)))
    except FileNotFoundError:
        pass
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None))
