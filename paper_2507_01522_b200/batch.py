"""Batched engine on the B200: the drop-in for the reference's BatchEnv.

Same constructor and methods as ``voltyard.engine.BatchEnv``
(engine.py:339-477): ``reset``, ``reseed``, ``step(actions, collect_infos)``,
``close``, ``action_size``, ``actions_per_slot``, ``obs_length``,
``observation_layout``.  Behind it the whole batch lives in HBM (PyTorch owns
every buffer; the C ABI borrows pointers, like CySimCore binds the engine's
memoryviews, _kernel.pyx:121-235) and one fused kernel launch advances every
env, including the auto-reset the reference runs as a Python loop
(engine.py:459-462).

Two calling conventions:
  * numpy in / numpy out (the reference's contract): actions are validated on
    the host exactly like engine.py:433-444, copied to the device, stepped, and
    obs / rewards / dones come back as detached host arrays.
  * torch CUDA tensors in / out (the throughput path): no host round trip; the
    returned tensors are the engine's output buffers, valid until the next
    step() or reset().  Out-of-range action indices are detected on the device
    and raised at the next synchronising call (``check_errors``).
"""

from __future__ import annotations

import ctypes as C
import math
import platform
import sys
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .envconfig import EnvConfig, ObsLayout
from .errors import EpisodeDone
from .exogenous import Dataset
from .station import StationTree
from .streams import PHASE_POLICY, split_seed, vstream_key
from .tables import StepTables, build_tables

BACKEND = "cuda"


def resolve_backend(name: str | None = None) -> str:
    """The product has exactly one backend (backends/__init__.py:30-40 shape)."""
    if name is None or name.lower() == BACKEND:
        return BACKEND
    raise ValueError(f"unknown backend {name!r}; this build provides only {BACKEND!r}")


def available_backends() -> tuple[str, ...]:
    return (BACKEND,)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class DeviceState:
    """Struct-of-arrays env state in HBM (vy_state).  Per-port tensors are [N, B]."""

    def __init__(self, B: int, n: int, device: torch.device):
        # leading dimension padded to whole 32-env warp tiles (vy_bind requires it)
        self.ld = ld = -(-B // 32) * 32
        self.B = B
        z = lambda *s, dt: torch.zeros(*s, dtype=dt, device=device)  # noqa: E731
        B = ld
        self.port_i = z(n, B, dt=torch.float64)
        self.port_soc = z(n, B, dt=torch.float64)
        self.port_de = z(n, B, dt=torch.float64)
        self.port_dtrem = z(n, B, dt=torch.int16)
        self.port_meta = z(n, B, dt=torch.uint8)
        self.step = z(B, dt=torch.int32)
        self.day = z(B, dt=torch.int32)
        self.episode = z(B, dt=torch.int32)
        self.env_seed = z(B, dt=torch.int64)  # uint64 bits
        self.akey = z(B, dt=torch.int64)
        self.b_i = z(B, dt=torch.float64)
        self.b_soc = z(B, dt=torch.float64)
        self.ep_profit = z(B, dt=torch.float64)
        self.ep_reward = z(B, dt=torch.float64)
        self.ep_missing = z(B, dt=torch.float64)
        self.ep_energy = z(B, dt=torch.float64)
        self.ep_overtime = z(B, dt=torch.int32)
        self.ep_declined = z(B, dt=torch.int32)
        self.ep_departures = z(B, dt=torch.int32)

    def ctypes(self, B: int) -> nat.VyState:
        s = nat.VyState()
        s.ld = self.ld
        for name, _ in nat.VyState._fields_[1:]:
            setattr(s, name, getattr(self, name).data_ptr())
        return s

    def bytes(self) -> int:
        return sum(v.numel() * v.element_size() for v in vars(self).values() if isinstance(v, torch.Tensor))

    def view(self, name: str) -> torch.Tensor:
        """Field without the warp-tile padding: [N, B] per port, [B] per env."""
        t = getattr(self, name)
        return t[..., : self.B]


class DeviceOutputs:
    """Per-step outputs (vy_outputs).  Info block is feature-major [k, B]."""

    def __init__(self, B: int, n: int, ns: int, obs_len: int, obs_dtype: torch.dtype, device: torch.device):
        self.device = device
        self.B, self.n, self.ns = B, n, ns
        self.ld = -(-B // 32) * 32
        self.obs = torch.zeros(B, obs_len, dtype=obs_dtype, device=device)
        self.reward = torch.zeros(B, dtype=obs_dtype, device=device)
        self.done = torch.zeros(B, dtype=torch.uint8, device=device)
        self.ep_stats = torch.zeros(8, self.ld, dtype=torch.float64, device=device)
        self.term_overtime = torch.zeros(self.ld, dtype=torch.int32, device=device)
        self.info = None

    def ensure_info(self) -> None:
        if self.info is not None:
            return
        B, n, ns, d = self.ld, self.n, self.ns, self.device
        f = lambda *s: torch.zeros(*s, dtype=torch.float64, device=d)  # noqa: E731
        i = lambda *s: torch.zeros(*s, dtype=torch.int32, device=d)  # noqa: E731
        self.info = dict(
            breakdown=f(10, B), flows=f(5, B), declined=i(B), arrivals_m=i(B), dep_n=i(B), dep_port=i(n, B),
            dep_overtime=i(n, B), dep_early=i(n, B), dep_pref=i(n, B), dep_missing=f(n, B), dep_cap=f(n, B),
            dep_soc=f(n, B), i_att=f(ns, B), i_used=f(ns, B), delivered=f(n, B), b_delivered=f(B))

    def ctypes(self) -> nat.VyOutputs:
        o = nat.VyOutputs()
        for name in ("obs", "reward", "done", "ep_stats", "term_overtime"):
            setattr(o, name, getattr(self, name).data_ptr())
        if self.info is not None:
            for name, t in self.info.items():
                setattr(o, name, t.data_ptr())
        return o


def _fresh(pin: torch.Tensor, dtype: torch.dtype) -> np.ndarray:
    """A new numpy array holding `pin` converted to `dtype` (the reference
    returns fresh copies, engine.py:463-464, so callers may keep them across
    steps); torch's CPU copy runs on all host threads."""
    out = torch.empty(pin.shape, dtype=dtype)
    out.copy_(pin)
    return out.numpy()


class BatchEnv:
    """B independent environments stepped in lockstep on one GPU.

    ``global_offset`` shifts the env index used for seeding (split_seed) and
    for the device RandomPolicy rows, so shards of a multi-GPU run are slices
    of one global batch (the worker-invariance contract, engine.py:1-8).
    """

    def __init__(self, config: EnvConfig, station: StationTree, dataset: Dataset, batch_size: int = 1,
                 master_seed: int = 0, env_seeds=None, auto_reset: bool = True, backend: str | None = None,
                 workers: int = 1, device=None, obs_dtype=torch.float32, global_offset: int = 0,
                 tables: StepTables | None = None):
        if batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if workers < 1:
            raise ValueError("workers must be >= 1")
        self.backend = resolve_backend(backend)
        self.config, self.station, self.dataset = config, station, dataset
        self.batch_size = B = int(batch_size)
        self.auto_reset = auto_reset
        self.workers = min(workers, batch_size)  # accepted for signature parity; results never depend on it
        self.global_offset = int(global_offset)
        if not torch.cuda.is_available():
            raise nat.NativeError("BatchEnv(backend='cuda') needs a CUDA device")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if obs_dtype not in (torch.float32, torch.float64):
            raise ValueError("obs_dtype must be torch.float32 or torch.float64")
        self.obs_dtype = obs_dtype
        # prebuilt tables: the reference plugin path receives the engine's KernelTables (plugin.py)
        self.tables: StepTables = tables if tables is not None else build_tables(config, station, dataset)
        t = self.tables
        if env_seeds is not None and len(env_seeds) != B:
            raise ValueError("env_seeds length must equal batch_size")
        self._lib = nat.lib()
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            nat.check(self._lib.vy_create(C.byref(t.as_ctypes()), B, self.device.index or 0, C.byref(h)), "vy_create")
        self._h = h
        self.states = DeviceState(B, t.n_ports, self.device)
        self.outs = DeviceOutputs(B, t.n_ports, t.n_slots, t.obs_len, obs_dtype, self.device)
        self._bind()
        self._act_buf = None
        self._host_act = None
        self._pins: dict = {}
        self._rings: dict = {}
        if env_seeds is None:
            self._seed_from_master(master_seed)
        else:
            self.set_env_seeds(env_seeds)
        self._needs_reset = True
        self._t = None  # common step counter while all envs move in lockstep
        self.profile_base = t.n_cat

    # -- plumbing ---------------------------------------------------------------

    @property
    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _bind(self) -> None:
        self._st_c = self.states.ctypes(self.batch_size)
        self._out_c = self.outs.ctypes()
        nat.check(self._lib.vy_bind(self._h, C.byref(self._st_c), C.byref(self._out_c)), "vy_bind")

    def _seed_from_master(self, master_seed: int) -> None:
        nat.check(self._lib.vy_seed_envs(self._h, int(master_seed), self.global_offset, self._stream),
                  "vy_seed_envs")

    def set_env_seeds(self, env_seeds) -> None:
        """Per-env seeds (uint64; BatchEnv(env_seeds=...), engine.py:371-374)."""
        if isinstance(env_seeds, np.ndarray) and env_seeds.dtype == np.uint64:
            seeds = np.ascontiguousarray(env_seeds)
        else:
            seeds = np.array([int(s) & ((1 << 64) - 1) for s in env_seeds], dtype=np.uint64)
        if seeds.shape != (self.batch_size,):
            raise ValueError("env_seeds length must equal batch_size")
        self.states.env_seed[: self.batch_size].copy_(torch.from_numpy(seeds.view(np.int64)).to(self.device))

    def set_outputs(self, obs: torch.Tensor | None = None, reward: torch.Tensor | None = None,
                    done: torch.Tensor | None = None) -> None:
        """Redirect the per-step obs / reward / done outputs into caller buffers
        (e.g. slices of a rollout buffer) so the kernel writes them in place."""
        B, L = self.batch_size, self.obs_length
        o = self.outs.ctypes()
        for name, t, shape, dt in (("obs", obs, (B, L), self.obs_dtype), ("reward", reward, (B,), self.obs_dtype),
                                   ("done", done, (B,), torch.uint8)):
            if t is None:
                continue
            if tuple(t.shape) != shape or t.dtype != dt or not t.is_contiguous() or t.device != self.device:
                raise ValueError(f"{name} buffer must be a contiguous {dt} tensor of shape {shape} on {self.device}")
            setattr(o, name, t.data_ptr())
        self._out_c = o
        nat.check(self._lib.vy_bind(self._h, C.byref(self._st_c), C.byref(self._out_c)), "vy_bind")

    def restore_outputs(self) -> None:
        self._bind()

    def _flags(self, infos: bool) -> int:
        f = nat.F_AUTO_RESET if self.auto_reset else 0
        if infos:
            f |= nat.F_INFOS
        if self.obs_dtype == torch.float64:
            f |= nat.F_OUT_F64
        return f

    # -- reference API properties (engine.py:386-403) ---------------------------

    @property
    def n_ports(self) -> int:
        return self.tables.n_ports

    @property
    def action_size(self) -> int:
        return self.tables.n_ports + 1

    @property
    def actions_per_slot(self) -> int:
        return 2 * self.tables.k + 1

    @property
    def obs_length(self) -> int:
        return self.tables.obs_len

    def observation_layout(self) -> ObsLayout:
        return ObsLayout(n_ports=self.tables.n_ports, horizon=self.tables.horizon)

    # -- API ----------------------------------------------------------------------

    def reseed(self, master_seed: int):
        self._seed_from_master(master_seed)
        self._needs_reset = True
        return self.reset()

    def reset(self, as_numpy: bool = True, injected_days=None):
        """First call starts episode 0, later calls advance every env (engine.py:414-424)."""
        mode = 0 if self._needs_reset else 1
        inj = None
        if injected_days is not None:
            inj = torch.as_tensor(np.asarray(injected_days, dtype=np.int32), device=self.device)
        nat.check(self._lib.vy_reset(self._h, None, mode, _ptr(inj), self._flags(False), self._stream), "vy_reset")
        self._needs_reset = False
        self._t = 0
        if not as_numpy:
            return self.outs.obs
        pin = self._pinned("obs", self.outs.obs)
        torch.cuda.current_stream(self.device).synchronize()
        return _fresh(pin, torch.float64)

    def _device_actions(self, actions) -> tuple[int, int, int, int, bool]:
        """-> (ptr, dtype code, row stride, col stride, host_path)."""
        B, A = self.batch_size, self.action_size
        if isinstance(actions, torch.Tensor) and actions.is_cuda:
            if tuple(actions.shape) != (B, A):
                raise ValueError(f"actions shape must be {(B, A)}, got {tuple(actions.shape)}")
            code = {torch.uint8: nat.VY_ACT_U8, torch.int32: nat.VY_ACT_I32, torch.int64: nat.VY_ACT_I64}.get(
                actions.dtype)
            if code is None:
                raise ValueError(f"unsupported action dtype {actions.dtype}")
            self._act_keep = actions
            return actions.data_ptr(), code, actions.stride(0), actions.stride(1), False
        a = np.ascontiguousarray(actions if not isinstance(actions, torch.Tensor) else actions.numpy(),
                                 dtype=np.int64)
        if a.shape != (B, A):
            raise ValueError(f"actions shape must be {(B, A)}, got {a.shape}")
        hi = 2 * self.tables.k
        # range check and narrowing cast with torch's multi-threaded CPU kernels
        # (numpy's are single-threaded: ~60 ms at B = 2^20)
        at = torch.from_numpy(a if a.flags.writeable else a.copy())
        lo_a, hi_a = torch.aminmax(at)
        if int(lo_a) < 0 or int(hi_a) > hi:
            raise ValueError(f"action indices must be in [0, {hi}]")
        small = hi <= 255
        if self._act_buf is None:
            dt = torch.uint8 if small else torch.int32
            self._act_buf = torch.empty(B, A, dtype=dt, device=self.device)
            self._host_act = torch.empty(B, A, dtype=dt, pin_memory=True)
        self._host_act.copy_(at)
        self._act_buf.copy_(self._host_act, non_blocking=True)
        code = nat.VY_ACT_U8 if small else nat.VY_ACT_I32
        return self._act_buf.data_ptr(), code, A, 1, True

    def step(self, actions, collect_infos: bool = True):
        """Step every env -> (obs, rewards, dones, infos); see module docstring."""
        if self._needs_reset:
            raise EpisodeDone("call reset() before step()")
        ptr, code, rs, cs, host = self._device_actions(actions)
        if not self.auto_reset and self._episode_over():
            raise EpisodeDone("an episode is done and auto_reset is off")
        if collect_infos and self.outs.info is None:
            self.outs.ensure_info()
            self._bind()
        rc = self._lib.vy_step(self._h, ptr, code, rs, cs, self._flags(collect_infos), None, self._stream)
        nat.check(rc, "vy_step")
        self._advance_clock()
        infos = self._build_infos() if collect_infos else None
        if host:
            if self.obs_dtype == torch.float64:
                # exact drop-in: D2H straight into pinned arrays handed to the caller
                obs = self._ring_out("obs", self.outs.obs)
                rew = self._ring_out("rew", self.outs.reward)
                done = self._ring_out("done", self.outs.done, np.bool_)
                self.check_errors()  # syncs the stream: the copies are complete
                return obs, rew, done, infos
            pins = [self._pinned(n, t) for n, t in (("obs", self.outs.obs), ("rew", self.outs.reward),
                                                     ("done", self.outs.done))]
            self.check_errors()  # syncs the stream: the copies into the pinned buffers are complete
            obs = _fresh(pins[0], torch.float64)
            rew = _fresh(pins[1], torch.float64)
            done = _fresh(pins[2], torch.bool)
            return obs, rew, done, infos
        return self.outs.obs, self.outs.reward, self.outs.done, infos

    def step_random(self, policy: "DeviceRandomPolicy", collect_infos: bool = False, keep_actions: bool = False,
                    device_counter: bool = False):
        """``step(policy.actions(obs))`` as ONE kernel: the RandomPolicy rows
        (policies.py:51-73) are drawn inside the step kernel (vy_step_random),
        bit-identical to ``policy.actions(env)`` followed by ``step``.  The
        throughput_probe loop body (engine.py:541-545).  With keep_actions the
        actions are also written to ``policy.last_actions`` (uint8 [B, n+1]);
        with device_counter the call index lives in device memory (graph
        replay; ``policy.calls`` is then advanced by the caller)."""
        if self._needs_reset:
            raise EpisodeDone("call reset() before step()")
        if policy.rows is not None and policy.rows != self.batch_size:
            raise ValueError("policy bound to a different batch size")
        if not self.auto_reset and self._episode_over():
            raise EpisodeDone("an episode is done and auto_reset is off")
        if collect_infos and self.outs.info is None:
            self.outs.ensure_info()
            self._bind()
        out = policy._buffer(self) if keep_actions else None
        counter = policy._device_counter(self) if device_counter else None
        rc = self._lib.vy_step_random(self._h, policy.seed & ((1 << 64) - 1), policy.index0,
                                      0 if device_counter else policy.calls, _ptr(counter), _ptr(out),
                                      self._flags(collect_infos), self._stream)
        nat.check(rc, "vy_step_random")
        if not device_counter:
            policy.calls += 1
        self._advance_clock()
        infos = self._build_infos() if collect_infos else None
        return self.outs.obs, self.outs.reward, self.outs.done, infos

    def step_injected(self, actions, draws, collect_infos: bool = False):
        """Step with arrival draws taken from ``draws`` (VY_F_INJECT).

        ``draws`` maps env -> list of (profile, stay, soc0, frac, pref) tuples;
        the count of tuples is the Poisson draw M of that env.
        """
        ptr, code, rs, cs, host = self._device_actions(actions)
        off, rows = [0], []
        for b in range(self.batch_size):
            cars = draws.get(b, []) if isinstance(draws, dict) else draws[b]
            rows.extend(cars)
            off.append(len(rows))
        cols = list(zip(*rows)) if rows else [[], [], [], [], []]
        dev = self.device
        bufs = dict(
            off=torch.tensor(off, dtype=torch.int32, device=dev),
            profile=torch.tensor(list(cols[0]) or [0], dtype=torch.uint8, device=dev),
            stay=torch.tensor(list(cols[1]) or [0], dtype=torch.int32, device=dev),
            soc0=torch.tensor(list(cols[2]) or [0.0], dtype=torch.float64, device=dev),
            frac=torch.tensor(list(cols[3]) or [0.0], dtype=torch.float64, device=dev),
            pref=torch.tensor(list(cols[4]) or [0], dtype=torch.uint8, device=dev))
        d = nat.VyDraws(**{k: v.data_ptr() for k, v in bufs.items()})
        if collect_infos and self.outs.info is None:
            self.outs.ensure_info()
            self._bind()
        flags = self._flags(collect_infos) | nat.F_INJECT
        nat.check(self._lib.vy_step(self._h, ptr, code, rs, cs, flags, C.byref(d), self._stream), "vy_step")
        torch.cuda.current_stream(dev).synchronize()
        self._advance_clock()
        return self.outs.obs, self.outs.reward, self.outs.done

    def _advance_clock(self) -> None:
        if self._t is None:
            return
        self._t += 1
        if self._t == self.tables.episode_steps and self.auto_reset:
            self._t = 0

    def _episode_over(self) -> bool:
        if self._t is not None:
            return self._t >= self.tables.episode_steps
        return bool((self.states.view("step") >= self.tables.episode_steps).any().item())

    def rollout(self, T: int, policy_seed: int, call0: int, obs_out: torch.Tensor, reward_out: torch.Tensor,
                done_out: torch.Tensor) -> None:
        """Fused T-step rollout with the device RandomPolicy (auto-reset on).

        obs_out: [T or 1, B, obs_len]; reward_out / done_out: [T or 1, B].  A
        leading dimension of 1 means every step overwrites the same buffer.
        """
        if self._needs_reset:
            raise EpisodeDone("call reset() before rollout()")
        if not self.auto_reset:
            raise ValueError("rollout() requires auto_reset=True")
        B, L = self.batch_size, self.obs_length
        ostride = 0 if obs_out.shape[0] == 1 else B * L
        rstride = 0 if reward_out.shape[0] == 1 else B
        if obs_out.dtype != self.obs_dtype or reward_out.dtype != self.obs_dtype or done_out.dtype != torch.uint8:
            raise ValueError("rollout buffers must match obs_dtype / uint8")
        flags = nat.F_AUTO_RESET | (nat.F_OUT_F64 if self.obs_dtype == torch.float64 else 0)
        rc = self._lib.vy_rollout(self._h, int(T), int(policy_seed) & ((1 << 64) - 1), self.global_offset,
                                  int(call0), obs_out.data_ptr(), ostride, reward_out.data_ptr(),
                                  done_out.data_ptr(), rstride, flags, self._stream)
        nat.check(rc, "vy_rollout")
        if self._t is not None:
            self._t = (self._t + T) % self.tables.episode_steps

    def _ring_out(self, name: str, t: torch.Tensor, view=None, depth: int = 4) -> np.ndarray:
        """Enqueue a D2H copy of `t` into a pinned host buffer and return it as
        a numpy array the caller owns.  The reference returns fresh copies
        (engine.py:463-464) so callers may keep them; buffers are drawn from a
        small ring and one is reused only once nothing but the ring refers to
        its array (a caller still holding the previous step's arrays keeps
        them intact), so the steady state allocates nothing and the copy lands
        at full DMA bandwidth with no second host pass."""
        ring = self._rings.setdefault(name, [])
        slot = None
        for cand in ring:
            # referents: the ring's list entry and getrefcount's argument
            if sys.getrefcount(cand[1]) <= 2:
                slot = cand
                break
        if slot is None:
            pin = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            arr = pin.numpy() if view is None else pin.numpy().view(view)
            slot = [pin, arr]
            if len(ring) < depth:
                ring.append(slot)
        slot[0].copy_(t, non_blocking=True)
        return slot[1]

    def _pinned(self, name: str, t: torch.Tensor) -> torch.Tensor:
        """Enqueue a D2H copy of `t` into a persistent pinned buffer (full DMA
        bandwidth; a pageable .cpu() goes through driver staging at a fraction)."""
        pin = self._pins.get(name)
        if pin is None or pin.shape != t.shape or pin.dtype != t.dtype:
            pin = self._pins[name] = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        pin.copy_(t, non_blocking=True)
        return pin

    def check_errors(self) -> None:
        """Raise ValueError if any kernel saw an out-of-range action index (syncs)."""
        word = C.c_uint32()
        nat.check(self._lib.vy_poll_error(self._h, 1, self._stream, C.byref(word)), "vy_poll_error")
        if word.value & 1:
            raise ValueError(f"action indices must be in [0, {2 * self.tables.k}]")

    def launch_count(self) -> int:
        return int(self._lib.vy_launch_count(self._h))

    def set_tiles_per_warp(self, k: int) -> None:
        """Shape the persistent step grid for a batch that shares the GPU with
        other batches (HeteroBatch): about k 32-env tiles per warp."""
        nat.check(self._lib.vy_set_tiles_per_warp(self._h, int(k)), "vy_set_tiles_per_warp")

    def set_wide(self, mode: int) -> None:
        """Small-batch kernel: 1 = one warp per env / one lane per port (low
        latency at small batches) for rollouts and for steps with uint8
        actions, 0 = one thread per env, -1 = by batch size (default: rollouts
        of <= 4096 envs go wide, steps stay on the tile kernel).  Outputs are
        identical either way (vy_set_wide)."""
        nat.check(self._lib.vy_set_wide(self._h, int(mode)), "vy_set_wide")

    def last_step_mode(self) -> int:
        """Step-kernel instantiation of the last step (1/2 lean, 0 generic; diagnostics)."""
        return int(self._lib.vy_last_step_mode(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            torch.cuda.synchronize(self.device)
            self._lib.vy_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- host views (reference layout) ---------------------------------------------

    def profile(self, p: int) -> tuple[float, float, float, float]:
        out = (C.c_double * 4)()
        nat.check(self._lib.vy_get_profile(self._h, int(p), out), "vy_get_profile")
        return tuple(out)

    def reference_state(self) -> dict:
        """State in the reference StateArrays layout (engine.py:221-279), numpy."""
        torch.cuda.synchronize(self.device)
        t = self.tables
        s = _Views(self.states)
        meta = s.port_meta.cpu().numpy().T.astype(np.int64)
        occ = (meta & 1).astype(np.int8)
        pref = ((meta >> 1) & 1).astype(np.int8)
        prof = meta >> 2
        # per-profile lookup tables (cap, r_ac, r_dc, tau), vectorised over [B, N]
        ids = np.unique(prof[occ == 1])
        lut = np.zeros((int(ids.max()) + 1 if ids.size else 1, 4))
        for p in ids:
            lut[int(p)] = self.profile(int(p))
        on = occ == 1
        dc = (np.asarray(t.kind)[None, :] == 1)
        cap = np.where(on, lut[prof, 0], 0.0)
        rbar = np.where(on, np.where(dc, lut[prof, 2], lut[prof, 1]), 0.0)
        tau = np.where(on, lut[prof, 3], 0.0)
        soc = s.port_soc.cpu().numpy().T.copy()
        with np.errstate(divide="ignore", invalid="ignore"):
            # charge_limit (vehicles.py:22-35) with the reference's operation order
            taper = (1.0 - soc) * rbar / (1.0 - tau)
        rhat = np.where(on, np.where(soc <= tau, rbar, taper), 0.0)
        b_soc = s.b_soc.cpu().numpy().copy()
        if t.battery_enabled:
            b_rhat = np.where(b_soc <= t.b_tau, t.b_rmax, (1.0 - b_soc) * t.b_rmax / (1.0 - t.b_tau))
        else:
            b_rhat = np.zeros_like(b_soc)
        return dict(
            occ=occ, pref=pref, i_drawn=s.port_i.cpu().numpy().T.copy(), soc=soc,
            de=s.port_de.cpu().numpy().T.copy(), dtrem=s.port_dtrem.cpu().numpy().T.astype(np.int64),
            cap=cap, rbar=rbar, tau=tau, rhat=rhat, b_i=s.b_i.cpu().numpy().copy(), b_soc=b_soc, b_rhat=b_rhat,
            step=s.step.cpu().numpy().astype(np.int64), day=s.day.cpu().numpy().astype(np.int64),
            episode=s.episode.cpu().numpy().astype(np.int64),
            env_seed=s.env_seed.cpu().numpy().view(np.uint64).copy(),
            ep_profit=s.ep_profit.cpu().numpy().copy(), ep_reward=s.ep_reward.cpu().numpy().copy(),
            ep_missing=s.ep_missing.cpu().numpy().copy(), ep_energy=s.ep_energy.cpu().numpy().copy(),
            ep_overtime=s.ep_overtime.cpu().numpy().astype(np.int64),
            ep_declined=s.ep_declined.cpu().numpy().astype(np.int64),
            ep_departures=s.ep_departures.cpu().numpy().astype(np.int64))

    def reference_outputs(self) -> dict:
        """Info block in the reference StepOutputs layout ([B, k], engine.py:282-336)."""
        torch.cuda.synchronize(self.device)
        B = self.batch_size
        o = {k: v[..., :B].cpu().numpy().T.copy() if v.dim() == 2 else v[:B].cpu().numpy().copy()
             for k, v in (self.outs.info or {}).items()}
        for k in ("declined", "arrivals_m", "dep_n", "dep_port", "dep_overtime", "dep_early", "dep_pref"):
            if k in o:
                o[k] = o[k].astype(np.int64)
        o["ep_stats"] = self.outs.ep_stats[:, :B].cpu().numpy().T.copy()
        o["term_overtime"] = self.outs.term_overtime[:B].cpu().numpy().astype(np.int64)
        return o

    def _build_infos(self) -> list:
        from .info import step_infos

        return step_infos(self)

    def inject_car(self, port: int, soc: float = 0.5, cap: float = 60.0, r_bar: float = 150.0, tau: float = 0.8,
                   de: float = 100.0, dtrem: int = 12, pref: int = 0, i_drawn: float = 0.0, b: int = 0) -> None:
        """Place a car directly into the device state (the reference's test
        fixture pattern, tests/helpers.py:163-189)."""
        p = int(self._lib.vy_add_profile(self._h, float(cap), float(r_bar), float(r_bar), float(tau)))
        if p < 0:
            raise ValueError(self._lib.vy_last_error().decode())
        s = self.states
        s.port_meta[port, b] = 1 | (int(pref) << 1) | (p << 2)
        s.port_i[port, b] = float(i_drawn)
        s.port_soc[port, b] = float(soc)
        s.port_de[port, b] = float(de)
        s.port_dtrem[port, b] = int(dtrem)


class _Views:
    """Attribute access to DeviceState fields without tile padding."""

    def __init__(self, st: DeviceState):
        self._st = st

    def __getattr__(self, name):
        return self._st.view(name)


class DeviceRandomPolicy:
    """RandomPolicy (policies.py:51-73) generated on the device.

    Row i draws from stream_key(seed, global_i, 2) exactly like the
    reference, so the action sequences are bit-identical.
    """

    def __init__(self, seed: int, n_ports: int, k: int):
        self.seed, self.n_ports, self.k = int(seed), n_ports, k
        self.index0 = 0
        self.rows = None
        self.calls = 0
        self._out = None

    def bind(self, env_indices) -> None:
        idx = list(env_indices)
        if idx and idx != list(range(idx[0], idx[0] + len(idx))):
            raise ValueError("device RandomPolicy binds a contiguous row range")
        self.index0 = idx[0] if idx else 0
        self.rows = len(idx)
        self.calls = 0

    def _buffer(self, env: BatchEnv) -> torch.Tensor:
        B = env.batch_size
        if self._out is None or self._out.shape[0] != B:
            self._out = torch.empty(B, self.n_ports + 1, dtype=torch.uint8, device=env.device)
        return self._out

    def _device_counter(self, env: BatchEnv) -> torch.Tensor:
        if getattr(self, "_counter", None) is None:
            # {call index, scratch}: see vy_random_actions_dev
            self._counter = torch.tensor([self.calls, 0], dtype=torch.int64, device=env.device)
        return self._counter

    @property
    def last_actions(self) -> torch.Tensor | None:
        """The uint8 [B, n+1] actions of the last actions() call (or
        BatchEnv.step_random(keep_actions=True))."""
        return self._out

    def actions(self, env: BatchEnv, device_counter: bool = False) -> torch.Tensor:
        """Next call's actions.  With device_counter the call index lives in
        device memory (graph-replayable); `calls` is then advanced by the caller."""
        B = env.batch_size
        if self.rows is not None and self.rows != B:
            raise ValueError("policy bound to a different batch size")
        self._buffer(env)
        if device_counter:
            rc = env._lib.vy_random_actions_dev(env._h, self.seed & ((1 << 64) - 1), self.index0,
                                                self._device_counter(env).data_ptr(), self._out.data_ptr(),
                                                env._stream)
            nat.check(rc, "vy_random_actions_dev")
            return self._out
        rc = env._lib.vy_random_actions(env._h, self.seed & ((1 << 64) - 1), self.index0, self.calls,
                                        self._out.data_ptr(), env._stream)
        nat.check(rc, "vy_random_actions")
        self.calls += 1
        return self._out


@dataclass(frozen=True)
class ThroughputReport:
    steps_per_second: float
    wall_seconds: float
    batch_size: int
    total_steps: int
    backend: str
    workers: int
    hardware: str

    def to_dict(self) -> dict:
        return dict(self.__dict__)


def hardware_fingerprint() -> str:
    name = torch.cuda.get_device_name() if torch.cuda.is_available() else platform.machine()
    return f"{name} | {platform.system()} {platform.release()} | python {platform.python_version()}"


def throughput_probe(config: EnvConfig, station: StationTree, dataset: Dataset, batch_size: int = 1,
                     total_steps: int = 100_000, seed: int = 0, backend: str | None = None,
                     workers: int = 1) -> ThroughputReport:
    """engine.py:515-556 on the device: random policy, auto-reset, infos off."""
    if total_steps < 1:
        raise ValueError("total_steps must be >= 1")
    env = BatchEnv(config, station, dataset, batch_size=batch_size, master_seed=seed, auto_reset=True,
                   backend=backend, workers=workers)
    pol = DeviceRandomPolicy(seed, env.n_ports, config.discretization_k)
    pol.bind(range(batch_size))
    env.reset(as_numpy=False)
    calls = -(-total_steps // batch_size)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(calls):
        env.step_random(pol)  # env.step(pol.actions(obs)) fused into one launch
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    env.close()
    return ThroughputReport(calls * batch_size / dt, dt, batch_size, calls * batch_size, BACKEND, workers,
                            hardware_fingerprint())


def policy_keys(seed: int, rows) -> np.ndarray:
    return vstream_key(seed, np.asarray(list(rows), dtype=np.int64), PHASE_POLICY)


__all__ = ["BatchEnv", "DeviceRandomPolicy", "ThroughputReport", "throughput_probe", "available_backends",
           "resolve_backend", "hardware_fingerprint", "split_seed", "math"]
