"""Summarize an ncu --csv launch list: per-kernel device time, DRAM bytes, and one apply's breakdown."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
    gi = hdr.index('Grid Size') if 'Grid Size' in hdr else None
    k = collections.OrderedDict()
    for r in data:
        d = k.setdefault(r[ii], {'name': r[ki], 'grid': r[gi] if gi is not None else ''})
        d[r[mi]] = float(r[vi].replace(',', ''))
    return list(k.values())


def short(d):
    nm = re.sub(r'\(.*', '', d['name']).replace('void ', '')[:34]
    ep = ' '.join(re.findall(r'[EG]\w+', d['name'])[:2])
    return f"{nm} {ep}"


if __name__ == "__main__":
    L = load(sys.argv[1])
    first, count = int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else len(L)
    tot = 0.0
    for d in L[first:first + count]:
        t = d['gpu__time_duration.sum'] / 1e3
        tot += t
        rd = d.get('dram__bytes_read.sum', 0) / 1e6
        wr = d.get('dram__bytes_write.sum', 0) / 1e6
        print(f"{t:9.1f} us  rd {rd:8.2f} MB wr {wr:7.2f} MB  {rd / max(t, 1e-9) * 1e-3 + wr / max(t, 1e-9) * 1e-3:6.2f} TB/s  "
              f"grid {d['grid']:>12}  {short(d)}")
    print(f"total {tot:.1f} us over {count} launches")
