import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1909_09825_b200 as fgt
for v in ([0.3, 0.5, 0.7, 0.9, 0.3], [0.9, 0.1, 0.5], list(np.random.default_rng(0).random(700)), [0.5,0.2]):
    try:
        p = fgt.plan(fgt.TransformRequest(v, [0.4], [1.0], 1.0), fgt.fold(fgt.cf_soe(8)))
        print("ok", len(v), p.target_perm[:5])
    except Exception as e:
        print("ERR", len(v), e)
