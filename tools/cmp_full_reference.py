import sys, json, time
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, golden_io as G
from oracle import oracle as O
from paper_2008_00326_b200.search import plan_search, assemble_result, result_to_json
dd, frame, models, cfg = G.full_scene()
plan = plan_search(frame, models, cfg)
print(plan.n)
which = sys.argv[1]
t0=time.time()
if which == 'oracle':
    out = O.run_plan(frame, models, plan, n_threads=8)
else:
    from paper_2008_00326_b200.engine import default_engine
    out = default_engine().run_plan(frame, models, plan)
print('run', time.time()-t0)
xy = G.world_xyyaw(frame, out.refined_cam)
d = xy - dd['xyyaw']; d[:,2] = (d[:,2] + np.pi) % (2*np.pi) - np.pi
close = (np.hypot(d[:,0], d[:,1]) <= 1e-4) & (np.abs(d[:,2]) <= 1e-4)
same = (out.j_o == dd['j_o']) & (out.j_r == dd['j_r'])
it = out.iterations == dd['reg_iters']
print('n0 eq', np.array_equal(out.n_first, dd['n0']), 'n1 eq', (out.n_rendered == dd['n1']).mean())
bad = sorted(set(np.nonzero(~close)[0].tolist()) | set(np.nonzero(~same)[0].tolist()))
print('close', close.sum(), 'same', same.sum(), 'iters', it.sum(), 'bad', len(bad), bad)
print('iters-bad', sorted(np.nonzero(~it)[0].tolist()))
print('n1-bad', sorted(np.nonzero(out.n_rendered != dd['n1'])[0].tolist()))
ref = json.loads(str(dd['result_json'])); mine = json.loads(result_to_json(assemble_result(plan, out, 0.0)))
for a,b in zip(ref['objects'], mine['objects']): print(a['object_id'], (a['proposal_index'],a['j_o'],a['j_r']) == (b['proposal_index'],b['j_o'],b['j_r']))
