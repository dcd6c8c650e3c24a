"""Column sums of a [M, N] bf16 gradient (the bias gradient of a linear
layer) on the device: torch's sum(0) vs a GEMM with a ones row."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200.ppo import colsum  # noqa: E402

M = 307200
for N in (360, 128, 64, 1):
    g = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
    ones = torch.ones(1, M, device="cuda", dtype=torch.bfloat16)
    fns = {"vy_colsum": lambda: colsum(g), "sum0": lambda: g.sum(0), "ones@g": lambda: ones @ g, "sum0_f32": lambda: g.sum(0, dtype=torch.float32)}
    ref = g.float().sum(0)
    for name, f in fns.items():
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            out = f()
        e.record()
        torch.cuda.synchronize()
        err = float((out.float().reshape(-1) - ref).abs().max() / ref.abs().max())
        print(f"N={N:4d} {name:9s} {s.elapsed_time(e) / 20 * 1e3:8.1f} us  rel err {err:.2e}")
