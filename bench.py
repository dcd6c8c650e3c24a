"""Benchmark: env-steps/s of the default 16-port station (BASELINE config C2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N)

Our arm.  A "step" is one pass of the throughput_probe loop body
(engine.py:541-545) over every env on the GPU: BatchEnv.step_random draws the
RandomPolicy rows inside the fused step kernel, which advances all envs
(auto-reset included) and emits obs/reward/done — one launch per step.  Each rank owns 2^20 envs
(weak scaling, global env indices rank*2^20 + i, so the union of shards is the
single-batch run); there is no data-path collective.  Time = max over ranks of
CUDA-event time around exactly K steps with barrier + synchronize on both
sides.  State + outputs are ~1.5 GB per rank, far above the 126 MB L2, so no
L2 flush is needed between steps.  All envs move through the 288-step day in
lockstep and the station load follows the arrival profile (empty at night,
~94% of ports occupied mid-afternoon), so the timed window is centred on
mid-day; the default K = 288 covers one whole day (every leg and both arms
use the same rule, see window_start).

Extra keys: roofline (the fused step on SURVEY §8(d)'s 1010 B/env-step, with
the ncu-measured DRAM bytes of the same day window as `traffic`), e2e (same metric
through the public API with host buffers: pinned actions H2D, step, obs /
reward / done D2H every step), cpu_baseline (the reference's own compiled
kernel from oracle/_ref — or the C oracle if it is absent — on the host's
cores, bounded sample), rollout (the fused T-step kernel, reported
separately), c4 (the 64-port battery station, config C4), ppo (C3), hetero
(C5), clocks (nvidia-smi sampled during the timed region).

Reference arm (--impl reference): the reference's compiled CPU kernel on all
host cores, one step = one env-step of a bounded 2^16-env sample of the same
workload over the same window of the day; rank 0 only.  Its line also carries
`api_level`: the reference's own throughput_probe (baseline/_ref) at B = 16 /
4096 x workers 1 / all cores, and config C1 literally.
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


# HBM throughput of plain read/write streams at the step kernel's mid-day
# mix (scripts/micro/rw_mix.cu, R:W = 3:5, profiles/r2_rw_mix.txt)
MIX_PEAK_GBS = 5821.0


def survey_bytes(t, T: int = 1) -> dict:
    """SURVEY.md §8(d) algorithmic bytes per env-step (the canonical roofline
    figure): minimal lossless SoA state S = 15 B/port + 44 B/env, read and
    written; uint8 actions N+1; float32 obs 4*obs_len; reward + done 5 B.
    N = 16: 2*284 + 17 + 420 + 5 = 1010 B (C2); C4: 3650 B.  The fused T-step
    rollout streams obs/reward/done every step and the state once:
    O + R + 2S/T (427 B at T = 288)."""
    S = 15 * t.n_ports + 44
    A = t.n_ports + 1
    O = 4 * t.obs_len
    return {"per_env_step": 2 * S + A + O + 5, "state": S, "actions": A, "obs": O, "reward_done": 5,
            "rollout_per_env_step": O + 5 + 2 * S / T}


def contract_bytes(t) -> dict:
    """Bytes one env-step of the fused step kernel moves under its own state
    layout: float64 i_drawn/soc/de + int16 dwell + uint8 meta
    per port (24 B of floats where §8(d)'s fp32 layout has 12: the price of
    bit-exact float64 state); per env int32 step/day, uint64 arrival key
    (read), float64 x4 + int32 x3 episode accumulators (read+write); actions
    uint8; obs float32; reward f32; done u8."""
    port = t.n_ports * (8 + 8 + 8 + 2 + 1)
    env_r = 4 + 4 + 8 + 4 * 8 + 3 * 4
    env_w = 4 + 4 * 8 + 3 * 4
    batt = 32 if t.battery_enabled else 0
    acts = t.n_ports + 1
    obs = 4 * t.obs_len
    total = 2 * port + env_r + env_w + batt + acts + obs + 4 + 1
    return {"per_env_step": total, "state_rw": 2 * port + env_r + env_w + batt, "actions": acts, "obs": obs,
            "reward_done": 5}


def window_traffic(steps: list[int], name: str = "r2_k_step_day_dram.json") -> tuple[float | None, str | None]:
    """Measured DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum, one
    ncu pass over every launch of a whole 288-step day of this workload,
    scripts/day_dram.sh) averaged over the day steps of the timed window."""
    path = os.path.join(ROOT, "profiles", name)
    if not os.path.exists(path):
        return None, None
    with open(path) as fh:
        per = json.load(fh)["bytes_per_launch_by_step"]
    return sum(per[s % len(per)] for s in steps) / len(steps), f"profiles/{name}"


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


def reference_api_rates(threads: int, budget_s: float = 4.0) -> dict | None:
    """The reference's own public API, unmodified, from baseline/_ref (pip
    install of /root/reference/pkg): throughput_probe (engine.py:515-556) with
    backend="compiled" at B = 16 and 4096, workers 1 and all host threads, and
    config C1 literally (16 envs x 288 steps, workers 1).  Each probe is sized
    to about `budget_s` seconds from a short calibration run."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "voltyard")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import voltyard
    from voltyard.config import default_setup as ref_setup
    from voltyard.engine import throughput_probe

    rc = ref_setup()
    out = {"source": "baseline/_ref voltyard.engine.throughput_probe(backend='compiled')", "cores": threads,
           "hardware": voltyard.engine.hardware_fingerprint(), "probes": []}
    for B, w in ((16, 1), (16, threads), (4096, 1), (4096, threads)):
        cal = throughput_probe(rc.env, rc.station, rc.dataset, batch_size=B, total_steps=B * 20, backend="compiled",
                               workers=w)
        total = max(B * 20, int(cal.steps_per_second * budget_s))
        rep = throughput_probe(rc.env, rc.station, rc.dataset, batch_size=B, total_steps=total, backend="compiled",
                               workers=w)
        out["probes"].append({"batch_size": B, "workers": w, "steps_per_s": rep.steps_per_second,
                              "total_steps": rep.total_steps, "seconds": rep.wall_seconds})
    # C1 literally: 16 envs x 288 steps (one whole episode), repeated
    reps = []
    for _ in range(3):
        rep = throughput_probe(rc.env, rc.station, rc.dataset, batch_size=16, total_steps=16 * 288,
                               backend="compiled", workers=1)
        reps.append(rep.steps_per_second)
    out["c1_literal"] = {"batch_size": 16, "steps": 288, "workers": 1, "steps_per_s": statistics.median(reps),
                         "repeats": len(reps)}
    return out


def run_reference_arm(args) -> None:
    """The reference's CPU implementation of the path on the box's host cores:
    its compiled kernel (oracle/_ref, built from the reference's own sources)
    over all host threads on a bounded 2^16-env sample of C2 over the same day
    window as our arm — the headline value; plus its public API
    (throughput_probe, baseline/_ref) at the §8(d) probe points."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2507_01522_b200 import default_setup

    rc = default_setup()
    threads = len(os.sched_getaffinity(0))
    B = 1 << 16
    w0 = window_start(args.steps, args.warmup) + args.warmup
    res = cpu_reference_rate(rc, B, w0, args.steps, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 default 16-port station, random actions (bounded CPU sample)",
                   "envs_per_step": B, "episode_steps": 288,
                   "timed_window": f"steps {w0}..{w0 + args.steps - 1} of the lockstep 288-step day "
                                   f"(same window as the GPU arm)"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_extras:
        api = reference_api_rates(threads)
        if api is not None:
            line["api_level"] = api
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=288)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=B_PER_GPU)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / rollout / PPO / C4 / C5 legs (profiling runs)")
    ap.add_argument("--ppo-iters", type=int, default=3, help="timed PPO iterations for the C3 leg (0 = skip)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2507_01522_b200 import default_setup
    from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy
    from paper_2507_01522_b200.workloads import c4_setup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        # one tiny collective so every rank's NCCL communicator is up (and logged) before timing
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)
        if rank == 0:
            print(f"[bench] NCCL communicator: nranks={int(t.item())} world={world}", file=sys.stderr, flush=True)

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

    stream = torch.cuda.current_stream()
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs")

    def timed_day_window(env, pol, K, W):
        """Advance to the window centred mid-day, W warm-up steps, then time
        exactly K fused steps (vy_step_random: RandomPolicy + step in one
        kernel) bracketed by barrier + synchronize; per-step CUDA events on the
        launching stream give the kernel's own average launch time."""
        advance = window_start(K, W, env.tables.episode_steps)
        for _ in range(advance + W):
            env.step_random(pol)
        barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = env.launch_count()
        t0.record(stream)
        for i in range(K):
            ev[i][0].record(stream)
            env.step_random(pol)
            ev[i][1].record(stream)
        t1.record(stream)
        barrier()
        steps = list(range(advance + W, advance + W + K))
        return (max_over_ranks(t0.elapsed_time(t1)), statistics.mean(s.elapsed_time(e) for s, e in ev),
                env.launch_count() - l0, steps)

    rc = default_setup()
    B = args.envs
    env = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=B, master_seed=0, global_offset=rank * B)
    pol = DeviceRandomPolicy(seed=0, n_ports=env.n_ports, k=rc.env.discretization_k)
    pol.bind(range(rank * B, rank * B + B))
    env.reset(as_numpy=False)
    with ClockSampler(local) as clocks:
        ms, step_kernel_ms, launches, wsteps = timed_day_window(env, pol, args.steps, args.warmup)
    value = args.steps * B * world / (ms / 1e3)

    # roofline of the dominant (only) kernel: the fused step, on SURVEY §8(d) bytes
    sb = survey_bytes(env.tables)
    cb = contract_bytes(env.tables)
    achieved = sb["per_env_step"] * B / (step_kernel_ms / 1e3) / 1e9
    traffic, tsrc = window_traffic(wsteps) if B == B_PER_GPU else (None, None)
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference synthetic generators: shopping/medium/eu, seed 0, 365 days)",
        "config": {"workload": "C2: default 16-port station (6 AC + 10 DC, multi_type), RandomPolicy actions, "
                               "288-step episodes with in-kernel auto-reset",
                   "envs_per_gpu": B, "global_envs": B * world, "episode_steps": rc.env.episode_steps,
                   "parallelism": f"env-sharded x{world}", "l2": "inputs ~1.5 GB/GPU >> 126 MB L2 (no flush)",
                   "obs_dtype": "f32", "state_dtype": "f64 (bit-exact with the reference)",
                   "step": "vy_step_random: RandomPolicy rows drawn inside the step kernel (one launch per step)",
                   "timed_window": f"steps {wsteps[0]}..{wsteps[-1]} of the lockstep {rc.env.episode_steps}-step "
                                   f"day (centred mid-day)"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "kernel": "vy::k_step<1> (fused RandomPolicy)", "kernel_ms": step_kernel_ms,
                     "bytes_per_env_step": sb["per_env_step"],
                     "bytes_note": "SURVEY §8(d): 2 x 284 B fp32 SoA state + 17 B u8 actions + 420 B f32 obs + 5 B",
                     "traffic_source": tsrc,
                     "traffic_per_env_step": traffic / B if traffic else None,
                     "traffic_frac": traffic / (step_kernel_ms / 1e3) / 1e9 / hbm if traffic else None,
                     "contract_f64": {"bytes_per_env_step": cb["per_env_step"],
                                      "frac": cb["per_env_step"] * B / (step_kernel_ms / 1e3) / 1e9 / hbm,
                                      "note": "the kernel's own float64-state contract (24 B of floats per port)"},
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not peaks.get("_fallback") else "fallback",
                     "mix_peak": {"gbs": MIX_PEAK_GBS,
                                  "traffic_frac": traffic / (step_kernel_ms / 1e3) / 1e9 / MIX_PEAK_GBS
                                  if traffic else None,
                                  "note": "plain 16-byte streams at the step's 0.37 R : 0.63 W DRAM mix "
                                          "(R:W = 3:5), profiles/r2_rw_mix.txt: the practical ceiling of "
                                          "the bytes the kernel moves; context only, frac uses peak"}},
        "clocks": clocks.summary(),
    }

    if not args.no_extras:
        # fused T-step rollout (state resident across T steps), reported separately
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
        rb = survey_bytes(env.tables, T)["rollout_per_env_step"]
        result["rollout"] = {"value": T * B * world / (rms / 1e3), "unit": UNIT, "T": T,
                             "ms": rms, "bytes_per_env_step": rb,
                             "achieved_gbs": rb * T * B / (rms / 1e3) / 1e9,
                             "frac": rb * T * B / (rms / 1e3) / 1e9 / hbm,
                             "note": "fused T-step kernel, in-kernel RandomPolicy, obs/reward/done every step; "
                                     "bytes = SURVEY §8(d) O + R + 2S/T"}

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
            env.step_random(pol)

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

        def pcie_ms() -> float:
            """The bus alone: the same D2H bytes with the H2D bytes concurrently, no kernel."""
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(e_steps):
                for h, d in zip(h_out[0], d_out[0]):
                    h.copy_(d, non_blocking=True)
                with torch.cuda.stream(copy_stream):
                    d_act.copy_(h_act, non_blocking=True)
            stream.wait_stream(copy_stream)
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / e_steps

        bus_ms = pcie_ms()
        result["e2e"] = {"value": e_steps * B * world / (ems / 1e3), "unit": UNIT,
                         "h2d_bytes_per_step": h_act.numel(),
                         "d2h_bytes_per_step": sum(t.numel() * t.element_size() for t in h_out[0]),
                         "serial_value": e_steps * B * world / (ems_serial / 1e3),
                         "pcie_bound": B * world / (bus_ms / 1e3),
                         "pcie_frac": (e_steps * B / (ems / 1e3)) / (B / (bus_ms / 1e3)),
                         "pcie_note": "pcie_bound: the same bytes copied alone (pinned D2H with the H2D concurrent), "
                                      "measured in this run",
                         "path": "BatchEnv.step with pinned host actions -> obs/reward/done to pinned host "
                                 "(two output sets, D2H on a copy stream overlapping the next step)"}
    env.close()

    if not args.no_extras and world == 1:
        # the public API call a reference user makes: throughput_probe (engine.py:515-556), wall clock,
        # one whole 288-step day of 2^20 envs from reset (device RandomPolicy fused into the step)
        from paper_2507_01522_b200.batch import throughput_probe

        rep = throughput_probe(rc.env, rc.station, rc.dataset, batch_size=B, total_steps=B * rc.env.episode_steps)
        result["api_probe"] = {"value": rep.steps_per_second, "unit": UNIT, "wall_seconds": rep.wall_seconds,
                               "total_steps": rep.total_steps, "batch_size": rep.batch_size,
                               "call": "throughput_probe(default_setup, batch_size=2^20, total_steps=288 * 2^20)",
                               "note": "wall clock incl. per-step host launch; the whole day from reset"}

    if not args.no_extras and world == 1:
        # config C1 (the reference's own CPU-runnable case: 16 envs x 288-step episodes) on the GPU: the fused
        # rollout on the small-batch kernel (one warp per env, one lane per port), one launch per episode
        c1 = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=16, master_seed=0)
        c1.reset(as_numpy=False)
        T1 = rc.env.episode_steps
        o1 = torch.empty(T1, 16, c1.obs_length, device=dev)
        r1 = torch.empty(T1, 16, device=dev)
        d1 = torch.empty(T1, 16, dtype=torch.uint8, device=dev)
        c1.rollout(T1, 0, 0, o1, r1, d1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        for rep in range(5):
            c1.rollout(T1, 0, (rep + 1) * T1, o1, r1, d1)
        ev[1].record(stream)
        torch.cuda.synchronize()
        c1ms = ev[0].elapsed_time(ev[1]) / 5
        result["c1"] = {"metric": METRIC, "value": 16 * T1 / (c1ms / 1e3), "unit": UNIT, "envs": 16, "T": T1,
                        "ms_per_episode": c1ms, "kernel": f"k_rollout_wide (mode {c1.last_step_mode()})",
                        "note": "config C1 on one B200: latency-bound (3 us per step of 16 envs); the reference "
                                "arm's api_level.c1_literal is the same workload on the host"}
        c1.close()

    if not args.no_extras:
        # config C4: 64 DC ports, 3-level splitter tree, battery, profit + satisfaction reward
        rc4 = c4_setup()
        B4 = 1 << 18
        env4 = BatchEnv(rc4.env, rc4.station, rc4.dataset, batch_size=B4, master_seed=0, global_offset=rank * B4)
        pol4 = DeviceRandomPolicy(seed=0, n_ports=env4.n_ports, k=rc4.env.discretization_k)
        pol4.bind(range(rank * B4, rank * B4 + B4))
        env4.reset(as_numpy=False)
        ms4, k4, _, w4 = timed_day_window(env4, pol4, args.steps, args.warmup)
        sb4 = survey_bytes(env4.tables)["per_env_step"]
        result["c4"] = {"metric": METRIC, "value": args.steps * B4 * world / (ms4 / 1e3), "unit": UNIT,
                        "envs_per_gpu": B4, "ms_per_step": ms4 / args.steps, "kernel_ms": k4,
                        "bytes_per_env_step": sb4, "frac": sb4 * B4 / (k4 / 1e3) / 1e9 / hbm,
                        "kernel_mode": env4.last_step_mode(),
                        "timed_window": f"steps {w4[0]}..{w4[-1]}",
                        "workload": "C4: 64 DC ports, nested_splitters 34-node tree, battery, highway/high/eu, "
                                    "sat0/sat1 penalties"}
        env4.close()

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
                         "optimizer_steps_per_100k_env_steps": 1e5 * cfg.update_epochs * cfg.n_minibatches
                                                               / (4096 * world * cfg.rollout_steps),
                         "rollout": tr.describe_rollout() if hasattr(tr, "describe_rollout") else None,
                         "update": tr.describe_update(),
                         "grad_allreduce": "NCCL all_reduce per minibatch" if world > 1 else "none (1 GPU)",
                         "paper_reference": "Chargax PPO(16) 0.65 s / 100k on RTX 4000 Ada (PAPER.md:239); a "
                                            "different workload (16 envs, 900-sample minibatches): see ppo_paper"}
        penv.close()
        if world == 1:
            # the paper's own PPO workload: Table 4 -- 12 vectorised envs, rollout 300
            # (batch 3600), 4 minibatches of 900, 4 epochs -- and the PPO(16) / PPO(1) rows' 16 and 1 envs
            #
            legs = {}
            for n_envs in (1, 12, 16):
                qenv = BatchEnv(rc.env, rc.station, rc.dataset, batch_size=n_envs, master_seed=1)
                qtr = PPOTrainer(qenv, PPOConfig(rollout_steps=300))
                qres = seconds_per_100k(qtr, 6, warmup=1)
                legs[f"envs_{n_envs}"] = {"value": qres["s_per_100k_steps"], "env_steps_per_s": qres["env_steps_per_s"],
                                          "minibatch": n_envs * 300 // 4, "timed_iterations": 6,
                                          "rollout": qtr.describe_rollout(), "update": qtr.describe_update()}
                qenv.close()
            result["ppo_paper"] = {"metric": "s per 100k PPO steps", "unit": "s", "higher_is_better": False,
                                   "legs": legs, "paper": {"PPO(16)": 0.65, "PPO(1)": 9.79, "hardware":
                                                           "RTX 4000 Ada (PAPER.md:239)"},
                                   "note": "same trainer as the ppo leg; at 1-16 envs the rollout is one vy_ppo_rollout "
                                           "launch and each minibatch three fused update kernels (CUDA graphs: one "
                                           "replay per rollout, one per update)"}

    if not args.no_extras:
        # config C5: 36 heterogeneous (region, scenario, traffic, station layout) groups sharing the GPU,
        # 2^20 envs per GPU (2^23 over 8 GPUs), device RandomPolicy per group
        from paper_2507_01522_b200.hetero import HeteroBatch, sweep_groups

        def hetero_rate(one_launch: bool) -> tuple[float, HeteroBatch]:
            hb = HeteroBatch(sweep_groups(B), master_seed=0, global_offset=rank * B, policy_seed=0)
            hb.reset()
            step = hb.graph_multi_step if one_launch else hb.graph_random_step
            hsteps = args.steps  # the same day window as the main leg (K = 288: one whole day)
            for _ in range(args.warmup + window_start(hsteps, args.warmup, rc.env.episode_steps)):  # centred mid-day
                step()
            barrier()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            for _ in range(hsteps):
                step()  # one CUDA-graph launch per heterogeneous step
            h1.record(stream)
            barrier()
            hms = max_over_ranks(h0.elapsed_time(h1))
            return hsteps * hb.total * world / (hms / 1e3), hb

        streams_value, hb = hetero_rate(False)
        kernels_streams = hb.kernels_per_step()
        hb.close()
        value, hb = hetero_rate(True)
        result["hetero"] = {"metric": METRIC, "value": value, "unit": UNIT,
                            "groups": len(hb.groups), "envs_per_gpu": hb.total, "global_envs": hb.total * world,
                            "kernels_per_step": 1, "graph_launches_per_step": 1,
                            "step": "k_step_multi: one persistent launch over all groups, per-tile config index, "
                                    "group Params in a constant-memory table, distinct table sets staged per CTA",
                            "multi": hb.multi_info(),
                            "per_group_streams": {"value": streams_value, "kernels_per_step": kernels_streams,
                                                  "note": "one fused step kernel per group on 12 streams, "
                                                          "one CUDA graph per step"},
                            "workload": "C5: regions x scenarios x traffic, single/multi/nested stations"}
        # roofline on SURVEY §8(d) bytes, per group (its station's port count / battery), env-weighted
        hbytes = sum(g.batch_size * survey_bytes(e.tables)["per_env_step"] for g, e in zip(hb.groups, hb.envs))
        avg_b = hbytes / hb.total
        result["hetero"]["roofline"] = {"bound": "hbm", "bytes_per_env_step": avg_b,
                                        "achieved": value / world * avg_b / 1e9, "peak": hbm, "unit": "GB/s",
                                        "frac": value / world * avg_b / 1e9 / hbm,
                                        "note": "SURVEY §8(d) bytes of each group's station, weighted by its envs"}
        hb.close()

    if rank == 0 and world == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        result["cpu_baseline"] = {k: v for k, v in cpu_reference_rate(
            rc, 1 << 16, wsteps[0], args.steps, threads).items() if k != "seconds"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


if __name__ == "__main__":
    main()
