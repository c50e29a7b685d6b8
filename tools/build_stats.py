"""Round/list/k2 counters of the fused builder (library built with
-DAK_BUILD_STATS): python tools/build_stats.py --n 1e8"""
import argparse, ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak
from paper_2106_12270_b200 import _lib
ap = argparse.ArgumentParser(); ap.add_argument("--n", type=float, default=1e8); ap.add_argument("--dist", default="uniform")
a = ap.parse_args(); n = int(a.n)
ws = ak.gen_uniform(n, ak.RngStream(seed=1), dtype=torch.float32, device="cuda") if a.dist == "uniform" else ak.gen_power_law(n, 1.0, ak.RngStream(seed=1), dtype=torch.float32, device="cuda")
L = _lib.lib()
wsb = torch.zeros(L.ak_build_workspace_bytes(n, 0), dtype=torch.uint8, device="cuda")
t = ak.AliasTable.empty(n, ws.total, torch.float32, "cuda")
_lib.check(L.ak_build_psa(_lib.ptr(ws.weights), 0, n, ws.total, _lib.ptr(t.rows), _lib.ptr(wsb), wsb.numel(), _lib.stream_ptr()))
torch.cuda.synchronize()
h = wsb[:32].cpu().view(torch.int32).tolist()
sections = (n + 511) // 512
print(f"sections {sections} rounds {h[2]} ({h[2]/sections:.2f}/sec) merge elems {h[3]} ({h[3]/n:.2f}/item) k2 {h[4]} lists {h[5]} ({h[5]/sections:.2f}/sec) useB {h[6]}")
