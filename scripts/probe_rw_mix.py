"""HBM throughput by read/write mix on this B200 (torch kernels over 2 GB):
write-only (fill), read-only (sum), copy (1 read : 1 write), and 1 read : 2
writes (one read stream, two output streams).  python scripts/probe_rw_mix.py"""
import torch

N = 1 << 28  # 2 GB of float64
a = torch.rand(N, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
c = torch.empty_like(a)


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


B = N * 8
for name, fn, nbytes in (("write only (fill)", lambda: b.fill_(1.0), B),
                         ("read only (sum)", lambda: a.sum(), B),
                         ("copy 1R:1W", lambda: b.copy_(a), 2 * B),
                         ("1R:2W (two outputs)", lambda: torch.stack([a, a], out=torch.empty(0)) if False else (b.copy_(a), c.copy_(a)), 4 * B)):
    ms = t(fn)
    print(f"{name:22s} {ms:7.3f} ms  {nbytes / ms / 1e6:7.1f} GB/s", flush=True)
a2 = a[: N // 2]
o1, o2 = b[: N // 2], c[: N // 2]


def one_read_two_writes():
    torch.mul(a2, 2.0, out=o1)
    torch.mul(a2, 3.0, out=o2)


ms = t(one_read_two_writes)
print(f"{'2x (1R:1W) half size':22s} {ms:7.3f} ms  {4 * (B // 2) / ms / 1e6:7.1f} GB/s")
