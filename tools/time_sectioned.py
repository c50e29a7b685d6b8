"""Time the bench's first sectioned sampling pass (N=1e9 f32 table, S=2^14,
RngStream(1, 7), <= 2^30 draws) for each library given, CUDA events, median
of --reps.  Variants are whole libaliaskit_b200.so builds loaded through
AK_LIB_PATH in a subprocess each:

    python tools/time_sectioned.py [lib.so ...] [--rng philox4x32|reference] [--dtype float64] [--S 8192]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(rng, reps, dtype, S):
    import numpy as np
    import torch
    sys.path.insert(0, ROOT)
    import paper_2106_12270_b200 as ak
    from paper_2106_12270_b200.sample import sectioned_sample_into
    N, M = 10**9, 10**11
    ws = ak.gen_uniform(N, ak.RngStream(seed=1), dtype=getattr(torch, dtype))
    t = ak.psa_construct(ws)
    del ws
    asg = ak.assign_sections(N, S, M, 1, 7)
    cd = torch.from_numpy(asg.counts).cuda()
    od = torch.from_numpy(np.concatenate([[0], np.cumsum(asg.counts)[:-1]])).cuda()
    k, tot = 0, 0
    while k < asg.n_sections and tot + int(asg.counts[k]) <= (1 << 30):
        tot += int(asg.counts[k])
        k += 1
    out = torch.empty(tot, dtype=torch.int64, device="cuda")
    r = ak.RngStream(1, 7)
    f = lambda: sectioned_sample_into(t, S, cd, od, 0, k, r, out, 0, rng)  # noqa: E731
    for _ in range(3):
        f()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    s = sorted(ts)[len(ts) // 2]
    chk = int(out[:: 1 << 16].sum().item())
    print(json.dumps(dict(lib=os.environ.get("AK_LIB_PATH", "default"), rng=rng, dtype=dtype, S=S, draws=tot, sections=k,
                          ms=s * 1e3, draws_per_s=tot / s, gbs=(tot * 8 + k * S * (8 if dtype == 'float32' else 16)) / s / 1e9, check=chk)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*")
    ap.add_argument("--rng", default="philox4x32")
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--S", type=int, default=1 << 14)
    a = ap.parse_args()
    if a.child:
        return child(a.rng, a.reps, a.dtype, a.S)
    for lib in a.libs or [""]:
        env = dict(os.environ)
        if lib:
            env["AK_LIB_PATH"] = os.path.abspath(lib)
        subprocess.run([sys.executable, __file__, "--child", "--rng", a.rng, "--reps", str(a.reps),
                        "--dtype", a.dtype, "--S", str(a.S)],
                       env=env, check=False)


if __name__ == "__main__":
    main()
