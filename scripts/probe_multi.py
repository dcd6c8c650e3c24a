"""C5 one-launch (k_step_multi) vs per-group stream launches over the bench's
mid-day window (steps 134..153), for the whole 36-group sweep and its fast-tree
and nested-splitter subsets.  python scripts/probe_multi.py [--subset all|fast|nested]"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--subset", default="all")
ap.add_argument("--B", type=int, default=1 << 20)
args = ap.parse_args()


def groups():
    gs = sweep_groups(args.B if args.subset == "all" else args.B * 3 // (2 if args.subset == "fast" else 1))
    if args.subset == "fast":
        gs = [g for i, g in enumerate(gs) if i % 3 != 2]
    elif args.subset == "nested":
        gs = [g for i, g in enumerate(gs) if i % 3 == 2]
    return gs


for one in (True, False):
    hb = HeteroBatch(groups(), master_seed=0, policy_seed=0)
    hb.reset()
    step = hb.graph_multi_step if one else hb.graph_random_step
    for _ in range(134):
        step()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(20):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    extra = hb.multi_info() if one else {}
    print(f"{args.subset:7s} {'one-launch' if one else 'streams':10s} envs {hb.total} {ms:.4f} ms/step "
          f"{hb.total / ms * 1e3:.3e} env-steps/s {extra}", flush=True)
    hb.close()
