"""Per-step kernel list of an ncu launch CSV (the launches between the last
two SGD kernels): count and total time per kernel.
usage: python tools/launch_step.py launches.csv [other.csv]"""
import collections
import csv
import sys


def step(path):
    rows = list(csv.reader(open(path)))
    hdr, seq = None, []
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get('Metric Name') != 'gpu__time_duration.sum':
            continue
        v = float(d['Metric Value'].replace(',', ''))
        u = d['Metric Unit']
        us = v / 1000 if u in ('ns', 'nsecond') else v if u in ('us', 'usecond') else v * 1000
        seq.append((d['Kernel Name'].split('(')[0].replace('void ', '')[:60], us))
    idx = [i for i, (k, _) in enumerate(seq) if 'sgd_kernel' in k]
    a, b = idx[-2], idx[-1]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, us in seq[a + 1:b + 1]:
        agg[k][0] += 1
        agg[k][1] += us
    return agg


def main():
    runs = [step(p) for p in sys.argv[1:]]
    keys = sorted(set().union(*runs), key=lambda k: -max(r.get(k, [0, 0])[1] for r in runs))
    for k in keys:
        print(f"{k:60s}" + "".join(f" {r.get(k, [0, 0])[0]:3d} {r.get(k, [0, 0])[1]:9.1f}"
                                    for r in runs))
    print(f"{'total':60s}" + "".join(f" {sum(v[0] for v in r.values()):3d} "
                                     f"{sum(v[1] for v in r.values()):9.1f}" for r in runs))


if __name__ == "__main__":
    main()
