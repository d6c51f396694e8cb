"""Summarise bench JSON lines and ncu launch lists from gpurun_out/ (dev helper)."""
import csv
import json
import sys
from collections import defaultdict


def bench(path):
    for l in open(path):
        if l.startswith('{'):
            d = json.loads(l)
            r = d.get('roofline', {})
            print(path, 'value', round(d['value']), 'ms/step', round(d['ms_per_step'], 4),
                  'e2e', d.get('e2e') and round(d['e2e']['value']), 'frac', r.get('frac') and round(r['frac'], 3),
                  'clk', d.get('clocks', {}).get('sm_mhz'))
            print('   layers', d.get('layers_ms_per_step'))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, defaultdict(list)
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out[(d['Kernel Name'][:90], d['Grid Size'])].append(float(d['Metric Value'].replace(',', '')))
    for k, v in out.items():
        print(len(v), 'avg us', round(sum(v) / len(v) / 1e3, 2), k)


for p in sys.argv[1:]:
    (launches if p.endswith('.csv') else bench)(p)
