"""k_step at a chosen step of the lockstep day (default 170: ~94% of ports
occupied, the slowest point), state restored before every timed launch so
each variant times the same transition.

  python scripts/probe_midday.py [--at 170] [--reps 25]
  python scripts/probe_midday.py --at 170 --ncu   # just advance + 1 step (for ncu --launch-skip)
"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import _native as nat, default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--at", type=int, default=170)
ap.add_argument("--reps", type=int, default=25)
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--fused", action="store_true", help="ncu mode: vy_step_random (RandomPolicy inside k_step)")
args = ap.parse_args()

rc = default_setup()
B = 1 << 20
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B)
pol = DeviceRandomPolicy(0, 16, 10)
pol.bind(range(B))
env.reset(as_numpy=False)
if args.ncu and args.fused:
    for _ in range(args.at + 1):
        env.step_random(pol)
    torch.cuda.synchronize()
    sys.exit(0)
for _ in range(args.at):
    env.step(pol.actions(env), collect_infos=False)
a = pol.actions(env)
if args.ncu:
    env.step(a, collect_infos=False)
    torch.cuda.synchronize()
    sys.exit(0)
snap = {k: v.clone() for k, v in vars(env.states).items() if isinstance(v, torch.Tensor)}
occ = float((env.states.port_meta[:, :B] & 1).float().mean())


def restore():
    for k, v in snap.items():
        getattr(env.states, k).copy_(v)


print(f"step {args.at}: occupancy {occ:.3f}")
for flags, name in ((1, "full"), (1 | 0x200, "memory-only"), (1 | 0x200 | 0x400 | 0x800, "loads only")):
    ts = []
    for _ in range(args.reps):
        restore()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        nat.check(env._lib.vy_step(env._h, a.data_ptr(), 0, 17, 1, flags, None, env._stream), "step")
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts = sorted(ts[3:])
    med = ts[len(ts) // 2]
    print(f"{name:12s} median ms {med:.4f}  eq GB/s {1414 * B / (med / 1e3) / 1e9:.0f}")
ts = []
for _ in range(args.reps):
    restore()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    nat.check(env._lib.vy_step_random(env._h, 0, 0, pol.calls - 1, None, None, 1, env._stream), "step_random")
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ts = sorted(ts[3:])
med = ts[len(ts) // 2]
print(f"{'fused policy':12s} median ms {med:.4f}  frac(1010 B) {1010 * B / (med / 1e3) / 1e9 / 6463.7:.3f}")
