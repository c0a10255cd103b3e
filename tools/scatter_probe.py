"""Cost of one random 8-byte scatter / gather per element on B200 (C5 size), against a
plain copy: the premise of a locality-reordered SpMV for the permuted C5 system."""
import torch
n = 4194304
g = torch.Generator(device="cuda").manual_seed(0)
perm = torch.randperm(n, device="cuda", generator=g)
x = torch.rand(n, device="cuda", dtype=torch.float64)
y = torch.empty_like(x)
idx32 = perm.to(torch.int32)
def t(f, reps=50):
    for _ in range(5): f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3
print("copy us", t(lambda: y.copy_(x)))
print("gather us", t(lambda: torch.index_select(x, 0, perm, out=y)))
print("scatter us", t(lambda: y.index_copy_(0, perm, x)))
print("gather sorted-idx us", t(lambda: torch.index_select(x, 0, torch.arange(n, device="cuda"), out=y)))
