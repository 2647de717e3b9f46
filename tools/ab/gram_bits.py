"""Write the GRAM solve's a_hat / history bytes for a few shapes (A/B of two
builds via BAK_LIB_PATH: the outputs must be bit-identical)."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_12570_b200 as pb  # noqa: E402

h = hashlib.sha256()
for seed, (obs, nv, dt, order) in enumerate([(50_000, 256, np.float64, "cyclic"), (70_001, 100, np.float32, "cyclic"),
                                              (33_333, 37, np.float64, "random"), (120_000, 200, np.float32, "random"),
                                              (5_000, 1, np.float64, "cyclic"), (9_999, 65, np.float64, "cyclic")]):
    rng = np.random.default_rng(seed)
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dt))
    if nv > 3:
        x[:, 2] = 0
    y = (x @ rng.uniform(-1, 1, nv).astype(dt) + 0.01 * rng.standard_normal(obs)).astype(dt)
    rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=7, tol=0, ordering=order, ordering_seed=3, record_history=True),
                       variant="gram")
    h.update(rep.a_hat.tobytes())
    h.update(np.asarray(rep.residual_norm_history).tobytes())
print(h.hexdigest())
