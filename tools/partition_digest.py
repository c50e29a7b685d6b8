"""SHA-256 digests of partition_items outputs (indices, weights, prefixes) on
fixed inputs, to compare two library builds bit for bit (AK_LIB_PATH)."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402

g = np.random.default_rng(3)
for n in (1, 7, 2048, 2049, 524288 + 5, 10**6 + 3, 10**8 + 11):
    for dt in (torch.float32, torch.float64):
        if n > 10**7:
            ws = ak.gen_uniform(n, ak.RngStream(seed=2), dtype=dt)
        else:
            w = g.pareto(1.2, n) + 1e-3
            ws = ak.make_weight_set(torch.from_numpy(w).to(dt).cuda())
        p = ak.partition_items(ws)
        h = hashlib.sha256()
        for t in (p.l_index, p.l_weight, p.h_index, p.h_weight, p.lprefix, p.hprefix):
            h.update(t.contiguous().cpu().numpy().tobytes())
        print(n, str(dt)[6:], h.hexdigest()[:16])
