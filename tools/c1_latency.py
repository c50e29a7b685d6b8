"""Wall-clock per public-API call at C1 size (N=1e6, M=1e6), host overhead included."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2106_12270_b200 as ak
w = torch.rand(10**6, device="cuda", dtype=torch.float64) + 1e-6
ws = ak.make_weight_set(w)
t = ak.psa_construct(ws)
out = torch.empty(10**6, dtype=torch.int64, device="cuda")
def wall(f, reps=200):
    for _ in range(10): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6
print("make_weight_set 1e6: %.1f us/call" % wall(lambda: ak.make_weight_set(w)))
print("psa_construct 1e6: %.1f us/call" % wall(lambda: ak.psa_construct(ws)))
print("sample_batch 1e6: %.1f us/call" % wall(lambda: ak.sample_batch(t, 10**6, ak.RngStream(1, 7), out=out)))
print("sectioned_sample 1e6 S=2^14: %.1f us/call" % wall(lambda: ak.sectioned_sample(t, 1 << 14, 10**6, ak.RngStream(1, 7))))
