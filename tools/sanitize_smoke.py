"""Small end-to-end exercise of every device entry point, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402

g = np.random.default_rng(11)
for n, kind in ((1, 0), (7, 0), (2049, 1), (70_001, 0), (70_001, 2), (60_000, 3)):
    if kind == 0:
        w = g.random(n) + 1e-6
    elif kind == 1:
        w = g.pareto(1.1, n) + 1e-6
    elif kind == 2:
        w = np.floor(g.random(n) * 5) + 1.0
    else:  # few deep lights among many barely-heavy items: multi-round pack sections
        light = g.random(n) < 0.1
        w = np.where(light, 1e-3 * (1 + g.random(n)), 1.1 + 0.01 * g.random(n))
    for dt in (torch.float64, torch.float32):
        ws = ak.make_weight_set(torch.from_numpy(w.astype(np.float32) if dt == torch.float32 else w).cuda())
        t = ak.psa_construct(ws)
        assert t.count_unwritten() == 0
        p = ak.partition_items(ws)
        plan = ak.compute_split_plan(p, min(7, n))
        ak.compute_split_plan(p, max(1, n // 16))  # many runs: TMA-staged windows
        ak.pack_section(p, plan, 1, ak.AliasTable.blank(n, ws.total, ws.dtype))
        tp = ak.psa_plus_construct(ws, block_size=64, threshold=4)
        assert tp.count_unwritten() == 0
        if n > 40_000:  # > 2048 blocks: several chunks in the residual-count scan
            tp = ak.psa_plus_construct(ws, block_size=16, threshold=2)
            assert tp.count_unwritten() == 0
        x = ak.sample_batch(t, 5000, ak.RngStream(3, 1), rng="reference")
        y = ak.sectioned_sample(t, 64, 5000, ak.RngStream(3, 2), rng="philox4x32")
        z = ak.sectioned_sample(t, 64, 5000, ak.RngStream(3, 2), rng="reference")
        ak.validate_table(t, ws)
        ak.frequency_counts(x, n)
        tq = ak.psa_plus_construct(ws)  # default block 4096 (bulk-copy staging when aligned)
        assert tq.count_unwritten() == 0
        ak.make_weight_set(ws.weights)
        if n > 1:
            hay = torch.sort(ws.weights.double())[0]
            ak.partial_pary_search(hay, hay[:: max(1, n // 100)].contiguous(), 8)
torch.cuda.synchronize()
print("sanitize smoke ok")
