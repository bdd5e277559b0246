"""Small end-to-end runs for compute-sanitizer: device set-up path (3-DoF + 6-DoF), flat path, batch."""
import sys, dataclasses
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import golden_io as G
from paper_2008_00326_b200 import estimate_poses, estimate_poses_many
from paper_2008_00326_b200.search import result_to_json
for name, over in (("c1_box_3dof", dict(dt=0.2)), ("c4_mixed_6dof", dict(viewpoints=4, n_inplane=2, max_proposals=None)),
                   ("c2_twocyl_color1", dict(dt=0.2)), ("c4_mixed_6dof", dict(max_proposals=60))):
    d, frame, models, cfg, _ = G.scene(name)
    cfg = dataclasses.replace(cfg, **over)
    r = estimate_poses(frame, models, cfg)
    print(name, r.proposals_evaluated, [e.proposal_index for e in r.estimates])
d, frame, models, cfg, _ = G.scene("c1_box_3dof")
rs = estimate_poses_many([(frame, models, dataclasses.replace(cfg, dt=0.2))] * 3, streams=2)
print("batch", [r.proposals_evaluated for r in rs])
