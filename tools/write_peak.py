"""Write-only HBM bandwidth probe (the lattice fill is a pure-write kernel): torch fill_ (a
vectorised store kernel) and cudaMemset over 8 GB, plus copy_ for reference; CUDA events,
best of 5 after a warm-up."""
import json

import torch


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


n = 1 << 30  # 8 GB fp64
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n // 2, dtype=torch.float64, device="cuda")
z = torch.empty(n // 2, dtype=torch.float64, device="cuda")
out = {}
ms = timeit(lambda: x.fill_(1.5))
out["fill_f64_gbs"] = 8 * n / ms / 1e6
ms = timeit(lambda: x.zero_())
out["zero_f64_gbs"] = 8 * n / ms / 1e6
ms = timeit(lambda: z.copy_(y))
out["copy_rw_gbs"] = 2 * 8 * (n // 2) / ms / 1e6
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
