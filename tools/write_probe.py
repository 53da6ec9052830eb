"""Write-only vs read-only vs copy HBM rates on this GPU (CUDA events, best of 10):
python tools/write_probe.py -- the ceiling of the write-dominated ops (prolongation)."""
import torch

n = 1 << 28  # 1 GiB of int32
a = torch.empty(n, dtype=torch.int32, device="cuda")
b = torch.empty(n, dtype=torch.int32, device="cuda")
a.fill_(1)


def best(fn, nbytes):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = 0.0
    for _ in range(10):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out = max(out, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return out


print({"write_fill_gbs": best(lambda: b.fill_(7), 4 * n),
       "write_zero_gbs": best(lambda: b.zero_(), 4 * n),
       "read_sum_gbs": best(lambda: a.sum(), 4 * n),
       "copy_gbs": best(lambda: b.copy_(a), 8 * n)})
