"""Phase timing of the fused PPO rollout (k_ppo_rollout): builds a variant of
the extension with -DVY_PPO_PROF (clock64 marks of CTA 0 thread 0) into
/tmp/vyprof, runs one rollout and prints the cycles per step of each phase.
python scripts/probe_ppo_phases.py [--envs 16] [--epc 4]"""
import argparse
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, ".")
ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=16)
ap.add_argument("--epc", type=int, default=0)
args = ap.parse_args()
if args.epc:
    os.environ["VY_PPO_EPC"] = str(args.epc)
from paper_2507_01522_b200 import _build, _native  # noqa: E402

out = Path("/tmp/vyprof")
out.mkdir(exist_ok=True)
objs = []
for src in _build._sources():
    o = out / (src.stem + ".o")
    subprocess.run([_build.nvcc(), *_build.NVCC_FLAGS, "-DVY_PPO_PROF", "-c", str(src), "-o", str(o)], check=True,
                   capture_output=True)
    objs.append(str(o))
lib = out / "libvoltyard_b200.so"
subprocess.run([_build.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib), *objs],
               check=True)
_native.LIB_PATH = lib

import torch  # noqa: E402

from paper_2507_01522_b200 import default_setup  # noqa: E402
from paper_2507_01522_b200.batch import BatchEnv  # noqa: E402
from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer  # noqa: E402

rc = default_setup()
env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=args.envs, master_seed=1)
T = 300
tr = PPOTrainer(env, PPOConfig(rollout_steps=T, use_graph=False))
tr.rollout()
torch.cuda.synchronize()
h = _native.lib()
h.vy_ppo_prof_read.argtypes = [C.c_void_p]
buf = (C.c_ulonglong * 16)()
h.vy_ppo_prof_read(buf)
names = ["env sync wait", "obs->A + sync", "L1 mma", "ep1 + sync", "L2 mma", "ep2 + sync", "L3 mma", "head + sync",
         "logp", "env step (warp 0)"]
tot = sum(buf[i] for i in range(10))
for i, nm in enumerate(names):
    print(f"{nm:20s} {buf[i] / T:8.0f} cyc/step  {100 * buf[i] / tot:5.1f}%")
print(f"total {tot / T:.0f} cycles per step")

h.vy_env_stamps_read.argtypes = [C.c_void_p]
st = (C.c_ulonglong * (256 * 16))()
h.vy_env_stamps_read(st)
import numpy as np  # noqa: E402

a = np.frombuffer(st, dtype=np.uint64).reshape(256, 16)[:, :9].astype(np.int64)
d = np.diff(a, axis=1)[1:]  # skip the first step (cold)
enames = ["frame+act+clip", "node sums", "charge", "flow sums", "dep sums", "arrivals", "reward+out", "obs"]
for i, nm in enumerate(enames):
    print(f"  env {nm:12s} mean {d[:, i].mean():7.0f}  median {np.median(d[:, i]):7.0f}  p90 {np.percentile(d[:, i], 90):7.0f}")
print(f"  env total mean {d.sum(1).mean():.0f}")
full = np.frombuffer(st, dtype=np.uint64).reshape(256, 16).astype(np.int64)[1:]
pre, fit = full[:, 9] - full[:, 1], full[:, 2] - full[:, 9]
print(f"  node sums before the rescale: mean {pre.mean():.0f}; rescale: mean {fit.mean():.0f}, "
      f"steps with a rescale {(fit > 200).mean() * 100:.0f}%")

# the fused update's gradient kernel: one update (16 minibatch launches), CTA 0 thread 0
tr.update()
torch.cuda.synchronize()
h.vy_upd_prof_read.argtypes = [C.c_void_p]
ub = (C.c_ulonglong * 16)()
h.vy_upd_prof_read(ub)
launches = tr.cfg.update_epochs * tr.cfg.n_minibatches
unames = ["stage issue + adv stats + row gather", "layer 1 + weights landed", "layers 2, head, value",
          "loss head + d logits", "backward to dz1", "weight gradients"]
utot = sum(ub[i] for i in range(6))
for i, nm in enumerate(unames):
    print(f"  grad {nm:38s} {ub[i] / launches:8.0f} cyc/launch  {100 * ub[i] / max(utot, 1):5.1f}%")
