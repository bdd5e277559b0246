"""Device (or C port) against tests/golden/c4f_full_reference.npz: python tools/cmp_full_reference_6dof.py device|oracle [stride]"""
import sys, json, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, golden_io as G, bench
from paper_2008_00326_b200.search import assemble_result, result_to_json
dd = G.load("c4f_full_reference")
which = sys.argv[1]; stride = int(sys.argv[2]) if len(sys.argv) > 2 else 1
frame, models, cfg, plan = bench.build_workload("c4", 1, 1, materialise_targets=(which == 'oracle'))
print(plan.n, len(dd['n0']))
idx = np.arange(0, plan.n, stride)
t0 = time.time()
if which == 'oracle':
    from oracle import oracle as O
    out = O.run_plan(frame, models, plan, index=idx, n_threads=8)
else:
    from paper_2008_00326_b200.engine import default_engine
    out = default_engine().run_plan(frame, models, plan, idx if stride > 1 else None)
print('run', time.time() - t0)
print('n0 eq', np.array_equal(out.n_first, dd['n0'][idx]))
same = (out.j_o == dd['j_o'][idx]) & (out.j_r == dd['j_r'][idx]) & (out.n_rendered == dd['n1'][idx])
it = out.iterations == dd['reg_iters'][idx]
print('same', same.sum(), 'of', idx.size, 'bad', idx[~same].tolist()[:80], 'iters-bad', idx[~it].tolist()[:80])
bad, badpose, iters = G.compare_with_full_reference_6dof(dd, out, idx)
print('costs/n1 differ', sorted(bad)); print('pose differ', sorted(badpose)); print('iters differ', sorted(iters))
if stride == 1:
    ref = json.loads(str(dd['result_json'])); mine = json.loads(result_to_json(assemble_result(plan, out, 0.0)))
    for a, b in zip(ref['objects'], mine['objects']): print(a['object_id'], (a['proposal_index'], a['j_o'], a['j_r']) == (b['proposal_index'], b['j_o'], b['j_r']))
