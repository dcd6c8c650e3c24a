"""Benchmark: env-steps/s of the default 16-port station (BASELINE config C2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N)

Our arm.  A "step" is one BatchEnv.step of every env on the GPU: the device
RandomPolicy writes uint8 actions, the fused step kernel advances all envs
(auto-reset included) and emits obs/reward/done.  Each rank owns 2^20 envs
(weak scaling, global env indices rank*2^20 + i, so the union of shards is the
single-batch run); there is no data-path collective.  Time = max over ranks of
CUDA-event time around exactly K steps with barrier + synchronize on both
sides.  State + outputs are ~1.5 GB per rank, far above the 126 MB L2, so no
L2 flush is needed between steps.  All envs move through the 288-step day in
lockstep and the station load follows the arrival profile (empty at night,
~94% of ports occupied mid-afternoon), so the timed window is centred on
mid-day; the default K = 288 covers one whole day (every leg and both arms
use the same rule, see window_start).

Extra keys: roofline (dominant kernel: the fused step), e2e (same metric
through the public API with host buffers: pinned actions H2D, step, obs /
reward / done D2H every step), cpu_baseline (the reference's own compiled
kernel from oracle/_ref — or the C oracle if it is absent — on the host's
cores, bounded sample), rollout (the fused T-step kernel, reported
separately), clocks (nvidia-smi sampled during the timed region).

Reference arm (--impl reference): the reference's compiled CPU kernel on all
host cores, one step = one env-step of a bounded 2^16-env sample of the same
workload over the same window of the day; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

B_PER_GPU = 1 << 20
METRIC = "env-steps/sec (whole box)"
UNIT = "env-steps/s"


def algorithmic_bytes(t) -> dict:
    """Bytes one env-step of the fused step kernel must move.

    State contract: float64 i_drawn/soc/de + int16 dwell + uint8 meta per port;
    per env int32 step/day, uint64 arrival key (read), float64 x4 + int32 x3
    episode accumulators (read+write); actions uint8; obs float32; reward f32;
    done u8.  The battery adds 2 x float64 read+write when enabled.
    """
    port = t.n_ports * (8 + 8 + 8 + 2 + 1)
    env_r = 4 + 4 + 8 + 4 * 8 + 3 * 4
    env_w = 4 + 4 * 8 + 3 * 4
    batt = 32 if t.battery_enabled else 0
    acts = t.n_ports + 1
    obs = 4 * t.obs_len
    total = 2 * port + env_r + env_w + batt + acts + obs + 4 + 1
    return {"per_env_step": total, "state_rw": 2 * port + env_r + env_w + batt, "actions": acts, "obs": obs,
            "reward_done": 5}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def window_start(steps: int, warmup: int, episode_steps: int = 288) -> int:
    """Untimed steps run before the warm-up so the timed window is centred on the
    middle of the 288-step day.  All envs move in lockstep through the day
    (reference semantics: every episode starts at step 0), and the station load
    follows the arrival profile: nearly empty at night, ~94% of ports occupied
    mid-afternoon (profiles/r1_day_profile.json).  K = 288 covers one whole day."""
    return max(0, (episode_steps - steps) // 2 - warmup)


def cpu_reference_rate(rc, B: int, advance: int, steps: int, threads: int, prefer_ref: bool = True) -> dict:
    """The reference's compiled kernel (oracle/_ref) or the C oracle on host cores,
    timed over the same window of the day as the GPU arm."""
    from oracle.harness import HostBatch, HostRandomPolicy, ref_available
    from paper_2507_01522_b200.tables import build_tables

    kind = "reference" if (prefer_ref and ref_available()) else "port"
    t = build_tables(rc.env, rc.station, rc.dataset)
    hb = HostBatch(t, B, master_seed=0, core="ref" if kind == "reference" else "oracle", threads=threads)
    pol = HostRandomPolicy(0, t.n_ports, t.k, range(B))
    hb.reset()
    for _ in range(advance):
        hb.core.step_all(pol.actions())
    acts = [pol.actions() for _ in range(steps)]
    t0 = time.perf_counter()
    for s in range(steps):
        hb.core.step_all(acts[s])
    dt = time.perf_counter() - t0
    return {"value": B * steps / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{B} envs x {steps} env-steps (steps {advance}..{advance + steps - 1} of the day) of the "
                      f"default station, core.step_range over {threads} threads, actions pre-generated",
            "seconds": dt}


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2507_01522_b200 import default_setup

    rc = default_setup()
    threads = len(os.sched_getaffinity(0))
    B = 1 << 16
    res = cpu_reference_rate(rc, B, window_start(args.steps, args.warmup) + args.warmup, args.steps, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 default 16-port station, random actions (bounded CPU sample)",
                   "envs_per_step": B, "episode_steps": 288,
                   "timed_window": f"steps {window_start(args.steps, args.warmup) + args.warmup}.."
                                   f"{window_start(args.steps, args.warmup) + args.warmup + args.steps - 1} of the "
                                   f"lockstep 288-step day (same window as the GPU arm)"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=288)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=B_PER_GPU)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / rollout / PPO legs (profiling runs)")
    ap.add_argument("--ppo-iters", type=int, default=3, help="timed PPO iterations for the C3 leg (0 = skip)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    rc = default_setup()
    B = args.envs
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=0, global_offset=rank * B)
    pol = DeviceRandomPolicy(seed=0, n_ports=env.n_ports, k=rc.env.discretization_k)
    pol.bind(range(rank * B, rank * B + B))
    env.reset(as_numpy=False)
    stream = torch.cuda.current_stream()
    advance = window_start(args.steps, args.warmup, rc.env.episode_steps)
    for _ in range(advance):
        env.step(pol.actions(env), collect_infos=False)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        env.step(pol.actions(env), collect_infos=False)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = env.launch_count()
    with ClockSampler(local) as clocks:
        t_start.record(stream)
        for i in range(args.steps):
            a = pol.actions(env)
            ev[i][0].record(stream)
            env.step(a, collect_infos=False)
            ev[i][1].record(stream)
        t_end.record(stream)
        barrier()
    launches = env.launch_count() - launches0
    ms = t_start.elapsed_time(t_end)
    ms_max = max_over_ranks(ms)
    step_kernel_ms = statistics.mean(s.elapsed_time(e) for s, e in ev)
    total_steps = args.steps * B * world
    value = total_steps / (ms_max / 1e3)

    # roofline of the dominant kernel (the fused step)
    ab = algorithmic_bytes(env.tables)
    peaks = load_peaks()
    achieved = ab["per_env_step"] * B / (step_kernel_ms / 1e3) / 1e9
    traffic = dram = None
    tpath = os.path.join(ROOT, "profiles", "step_kernel_dram_bytes.json")
    if os.path.exists(tpath) and B == B_PER_GPU and args.steps == 288:
        # dram__bytes_read.sum + dram__bytes_write.sum per k_step launch, averaged over
        # the 288 launches of this same day window (ncu, scripts/day_dram.sh).  The
        # kernel neither reads nor rewrites ports that are empty in a whole 32-env
        # tile, so its real traffic is below the step contract's 1414 B/env-step;
        # dram_frac is that real traffic over the measured time.
        with open(tpath) as fh:
            traffic = json.load(fh).get("bytes_per_launch")
        dram = {"bytes_per_env_step": traffic / B, "achieved": traffic / (step_kernel_ms / 1e3) / 1e9,
                "frac": traffic / (step_kernel_ms / 1e3) / 1e9 / peaks.get("hbm_gbs"),
                "source": "profiles/step_kernel_dram_bytes.json"}

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference synthetic generators: shopping/medium/eu, seed 0, 365 days)",
        "config": {"workload": "C2: default 16-port station (6 AC + 10 DC, multi_type), random actions, "
                               "288-step episodes with in-kernel auto-reset",
                   "envs_per_gpu": B, "global_envs": B * world, "episode_steps": rc.env.episode_steps,
                   "parallelism": f"env-sharded x{world}", "l2": "inputs ~1.5 GB/GPU >> 126 MB L2 (no flush)",
                   "obs_dtype": "f32", "actions": "u8 from device RandomPolicy",
                   "timed_window": f"steps {advance + args.warmup}..{advance + args.warmup + args.steps - 1} "
                                   f"of the lockstep {rc.env.episode_steps}-step day (centred mid-day)"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                     "frac": achieved / peaks.get("hbm_gbs"), "traffic": traffic,
                     "kernel": "vy::k_step", "kernel_ms": step_kernel_ms,
                     "bytes_per_env_step": ab["per_env_step"],
                     "bytes_note": "step contract: full f64 port state read + written, u8 actions, f32 obs",
                     "dram": dram,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not peaks.get("_fallback") else "fallback"},
        "clocks": clocks.summary(),
    }

    if not args.no_extras:
        # fused T-step rollout (state in registers), reported separately
        T = rc.env.episode_steps
        obs_b = torch.empty(1, B, env.obs_length, device=dev)
        rew_b = torch.empty(1, B, device=dev)
        done_b = torch.empty(1, B, dtype=torch.uint8, device=dev)
        env.rollout(8, 0, pol.calls, obs_b, rew_b, done_b)
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        env.rollout(T, 0, pol.calls + 8, obs_b, rew_b, done_b)
        s1.record(stream)
        barrier()
        rms = max_over_ranks(s0.elapsed_time(s1))
        rb = ab["obs"] + ab["reward_done"] + 2 * ab["state_rw"] / T
        result["rollout"] = {"value": T * B * world / (rms / 1e3), "unit": UNIT, "T": T,
                             "ms": rms, "bytes_per_env_step": rb,
                             "achieved_gbs": rb * T * B / (rms / 1e3) / 1e9,
                             "note": "fused T-step kernel, in-kernel RandomPolicy, obs/reward/done every step"}

        # e2e through the public API with host buffers: every step copies its
        # actions H2D from pinned memory and its obs / reward / done D2H to pinned
        # memory.  Pipelined the way a host consumer would run it: the step
        # writes one of two output sets (BatchEnv.set_outputs) while a copy
        # stream drains the other, so the PCIe D2H of step t overlaps the H2D
        # and kernel of step t+1 (the bus is the bound: ~463 MB per step).
        # The serial variant (one stream) is reported alongside.
        h_act = torch.empty(B, env.action_size, dtype=torch.uint8, pin_memory=True)
        h_act.copy_(pol.actions(env).cpu())
        d_act = torch.empty_like(h_act, device=dev)
        L = env.obs_length
        d_out = [(torch.empty(B, L, device=dev), torch.empty(B, device=dev),
                  torch.empty(B, dtype=torch.uint8, device=dev)) for _ in range(2)]
        h_out = [(torch.empty(B, L, pin_memory=True), torch.empty(B, pin_memory=True),
                  torch.empty(B, dtype=torch.uint8, pin_memory=True)) for _ in range(2)]
        copy_stream = torch.cuda.Stream(device=dev)
        e_steps = max(3, min(args.steps, 20))
        while env._t != window_start(e_steps, 2, rc.env.episode_steps):  # centre this window mid-day too
            env.step(pol.actions(env), collect_infos=False)

        def e2e_run(pipelined: bool) -> float:
            written = [torch.cuda.Event() for _ in range(2)]
            drained = [None, None]
            e0 = None
            for i in range(e_steps + 2):
                if i == 2:
                    torch.cuda.synchronize()
                    barrier()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                k = i % 2 if pipelined else 0
                if drained[k] is not None:
                    stream.wait_event(drained[k])  # set k's previous D2H has finished reading it
                d_act.copy_(h_act, non_blocking=True)
                env.set_outputs(*d_out[k])
                env.step(d_act, collect_infos=False)
                written[k].record(stream)
                cs = copy_stream if pipelined else stream
                cs.wait_event(written[k])
                with torch.cuda.stream(cs):
                    for h, d in zip(h_out[k], d_out[k]):
                        h.copy_(d, non_blocking=True)
                    drained[k] = torch.cuda.Event()
                    drained[k].record(cs)
            e1 = torch.cuda.Event(enable_timing=True)
            stream.wait_stream(copy_stream)
            e1.record(stream)
            barrier()
            return max_over_ranks(e0.elapsed_time(e1))

        ems_serial = e2e_run(False)
        ems = e2e_run(True)
        env.restore_outputs()
        result["e2e"] = {"value": e_steps * B * world / (ems / 1e3), "unit": UNIT,
                         "h2d_bytes_per_step": h_act.numel(),
                         "d2h_bytes_per_step": sum(t.numel() * t.element_size() for t in h_out[0]),
                         "serial_value": e_steps * B * world / (ems_serial / 1e3),
                         "path": "BatchEnv.step with pinned host actions -> obs/reward/done to pinned host "
                                 "(two output sets, D2H on a copy stream overlapping the next step)"}

    if not args.no_extras and args.ppo_iters > 0:
        # config C3: PPO with 4096 envs per GPU, Table 4 hyperparameters,
        # gradients all-reduced over NCCL when world > 1
        from paper_2507_01522_b200.ppo import PPOConfig, PPOTrainer, seconds_per_100k

        penv = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=4096, master_seed=1, global_offset=rank * 4096)
        cfg = PPOConfig(rollout_steps=300)
        tr = PPOTrainer(penv, cfg)
        res = seconds_per_100k(tr, args.ppo_iters, warmup=1)
        result["ppo"] = {"metric": "s per 100k PPO steps", "value": res["s_per_100k_steps"],
                         "env_steps_per_s": res["env_steps_per_s"], "envs_per_gpu": 4096,
                         "rollout_steps": cfg.rollout_steps, "epochs": cfg.update_epochs,
                         "minibatches": cfg.n_minibatches, "hidden": cfg.hidden, "timed_iterations": args.ppo_iters,
                         "rollout": "CUDA graph (policy fwd bf16: 3 GEMMs with block-diagonal layer 2 and merged heads + vy_ppo_sample_rng Gumbel-max kernel with in-kernel uniforms + k_step) x 300",
                         "update": ("one CUDA graph per update on 1 GPU (eager with the all-reduce): vy_gae, "
                                    "vy_gather_rows minibatch gather, bf16 GEMMs at 8-aligned widths with column-sum bias "
                                    "gradients (vy_colsum), vy_ppo_head_fwd/_bwd fused log-prob/entropy head, fused Adam"),
                         "grad_allreduce": "NCCL all_reduce(AVG) per minibatch" if world > 1 else "none (1 GPU)",
                         "paper_reference": "Chargax PPO(16) 0.65 s / 100k on RTX 4000 Ada (PAPER.md:239)"}
        penv.close()

    if not args.no_extras:
        # config C5: 36 heterogeneous (region, scenario, traffic, station layout) groups sharing the GPU,
        # 2^20 envs per GPU (2^23 over 8 GPUs), device RandomPolicy per group
        from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups

        hb = HeteroBatch(sweep_groups(B), master_seed=0, global_offset=rank * B, policy_seed=0)
        hb.reset()
        hsteps = args.steps  # the same day window as the main leg (K = 288: one whole day)
        for _ in range(3 + window_start(hsteps, 3, rc.env.episode_steps)):  # window centred mid-day
            hb.graph_random_step()
        barrier()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = sum(e.launch_count() for e in hb.envs)
        h0.record(stream)
        for _ in range(hsteps):
            hb.graph_random_step()  # one CUDA-graph launch per heterogeneous step
        h1.record(stream)
        barrier()
        hms = max_over_ranks(h0.elapsed_time(h1))
        result["hetero"] = {"metric": METRIC, "value": hsteps * hb.total * world / (hms / 1e3), "unit": UNIT,
                            "groups": len(hb.groups), "envs_per_gpu": hb.total, "global_envs": hb.total * world,
                            "kernels_per_step": 2 * len(hb.groups), "graph_launches_per_step": 1,
                            "workload": "C5: regions x scenarios x traffic, single/multi/nested stations"}
        hb.close()

    if rank == 0 and world == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        result["cpu_baseline"] = {k: v for k, v in cpu_reference_rate(
            rc, 1 << 16, advance + args.warmup, args.steps, threads).items() if k != "seconds"}
    env.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


if __name__ == "__main__":
    main()
