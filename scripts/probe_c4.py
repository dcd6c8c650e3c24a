"""Config C4 (64 DC ports, 34-node tree, battery) at a chosen step of the
lockstep day: k_step time (state restored before each timed launch), or with
--ncu just advance and run one fused step for ncu --launch-skip.

  python scripts/probe_c4.py [--at 144] [--B 262144] [--ncu]"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402
from paper_2507_01522_b200.workloads import c4_setup  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--at", type=int, default=144)
ap.add_argument("--B", type=int, default=1 << 18)
ap.add_argument("--reps", type=int, default=15)
ap.add_argument("--ncu", action="store_true")
args = ap.parse_args()
rc = c4_setup()
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=args.B)
pol = DeviceRandomPolicy(0, env.n_ports, rc.env.discretization_k)
pol.bind(range(args.B))
env.reset(as_numpy=False)
for _ in range(args.at):
    env.step_random(pol)
torch.cuda.synchronize()
if args.ncu:
    env.step_random(pol)
    torch.cuda.synchronize()
    sys.exit(0)
snap = {k: v.clone() for k, v in vars(env.states).items() if isinstance(v, torch.Tensor)}
ts = []
for _ in range(args.reps):
    for k, v in snap.items():
        getattr(env.states, k).copy_(v)
    calls = pol.calls
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    env.step_random(pol)
    e.record()
    torch.cuda.synchronize()
    pol.calls = calls
    env._t = args.at
    ts.append(s.elapsed_time(e))
ts = sorted(ts[2:])
med = ts[len(ts) // 2]
print(f"C4 step {args.at}: {med:.4f} ms  {args.B / med * 1e3:.3e} env-steps/s  frac(3650 B) "
      f"{3650 * args.B / (med / 1e3) / 1e9 / 6458:.3f}  mode {env.last_step_mode()}")
