import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from golden_io import load, table, config_from_case
from paper_2604_00510_b200.engine import Engine

name = sys.argv[1] if len(sys.argv) > 1 else 'c1_M256'
case = next(c for c in load('waves') if c['name'] == name)
recs = load('workloads')[case['workload']][: len(case['outcomes'])]
cfg = config_from_case(case)
n = len(recs)

def run(pipe, upto):
    os.environ['TS_NO_PIPELINE'] = '0' if pipe else '1'
    os.environ['TS_PIPELINE_SYNC'] = os.environ.get('SYNC', '0')
    eng = Engine(cfg, 0)
    eng.load(table(recs, case['arrival_steps']))
    counts = torch.zeros(3, dtype=torch.int64, device='cuda')
    rec = torch.zeros(n * 16, dtype=torch.uint8, device='cuda')
    for step in range(upto):
        eng.step_counts(step, counts.data_ptr()); eng.step_admit(step, counts.data_ptr(), 1, 0)
        eng.step_records(step, rec.data_ptr()); eng.step_targets(step, rec.data_ptr())
        tg = eng.read_targets()
        eng.step_wave(step)
    return eng, tg

for upto in range(1, case['steps'] + 1):
    a, ta = run(True, upto); b, tb = run(False, upto)
    bad = []
    for i in range(n):
        x, y = a.tree(i), b.tree(i)
        if len(x['parent']) != len(y['parent']) or any((x[k] != y[k]).any() for k in x if len(x[k]) == len(y[k])):
            bad.append(i)
    print('after wave', upto - 1, 'targets', [t for t in tb if t >= 8][:10], 'diff searches', bad[:10])
    if bad:
        i = bad[0]
        x, y = a.tree(i), b.tree(i)
        m = min(len(x['parent']), len(y['parent']))
        print(' search', i, 'target', tb[i], 'nodes pipe', len(x['parent']), 'seq', len(y['parent']))
        for k in x:
            d = np.nonzero(x[k][:m] != y[k][:m])[0]
            if d.size: print('  field', k, 'first diff node', d[0], 'pipe', x[k][d[0]], 'seq', y[k][d[0]])
        break
