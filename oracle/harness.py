"""CPU oracle harness (TEST INFRASTRUCTURE ONLY).

``HostBatch`` reproduces the reference BatchEnv semantics (engine.py:339-477:
reset episode numbering, validation, auto-reset of done rows, detached
copies) over numpy arrays in the reference layout (engine.py:221-336), with a
pluggable CPU stepping core:

  core="oracle"  the plain-C restatement oracle/vy_oracle.c (always present)
  core="ref"     the reference's own compiled Cython kernel, built from
                 /root/reference by oracle/build_ref.py into oracle/_ref/

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs import this module, and only as the checker.
"""

from __future__ import annotations

import ctypes as C
import importlib.util
import subprocess
import sysconfig
from pathlib import Path
from types import SimpleNamespace

import numpy as np

from paper_2507_01522_b200.errors import EpisodeDone
from paper_2507_01522_b200.streams import PHASE_POLICY, split_seed, vstream_key
from paper_2507_01522_b200.tables import StepTables

HERE = Path(__file__).resolve().parent
LIB = HERE / "lib" / "libvy_oracle.so"
REF = HERE / "_ref" / f"_kernel{sysconfig.get_config_var('EXT_SUFFIX')}"

_P = C.c_void_p


class _State(C.Structure):
    _fields_ = [(n, _P) for n in (
        "occ", "pref", "i_drawn", "soc", "de", "cap", "rbar", "tau", "rhat", "dtrem", "b_i", "b_soc", "b_rhat",
        "step", "day", "episode", "env_seed", "ep_profit", "ep_reward", "ep_missing", "ep_energy",
        "ep_overtime", "ep_declined", "ep_departures")]


class _Outs(C.Structure):
    _fields_ = [(n, _P) for n in (
        "obs", "reward", "done", "breakdown", "flows", "declined", "arrivals_m", "dep_n", "dep_port",
        "dep_missing", "dep_overtime", "dep_early", "dep_pref", "dep_cap", "dep_soc", "term_overtime",
        "ep_stats", "i_att", "i_used", "delivered", "b_delivered", "scratch")]


_lib = None


def load_oracle() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        lib = C.CDLL(str(LIB))
        lib.vyo_reset_env.argtypes = [_P, _P, _P, C.c_int64, C.c_int64]
        lib.vyo_step_range.argtypes = [_P, _P, _P, C.c_int64, C.c_int64, _P]
        lib.vyo_step_parallel.argtypes = [_P, _P, _P, C.c_int64, _P, C.c_int]
        lib.vyo_random_actions.argtypes = [_P, C.c_int64, C.c_int32, C.c_int32, _P]
        lib.vyo_reset_parallel.argtypes = [_P, _P, _P, C.c_int64, C.c_int, C.c_int]
        lib.vyo_step_parallel_autoreset.argtypes = [_P, _P, _P, C.c_int64, _P, C.c_int]
        lib.vyo_random_actions_parallel.argtypes = [_P, C.c_int64, C.c_int32, C.c_int32, _P, C.c_int]
        _lib = lib
    return _lib


def ref_available() -> bool:
    return REF.exists()


def _load_ref():
    spec = importlib.util.spec_from_file_location("_kernel", REF)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def allocate_state(B: int, n: int, seeds) -> SimpleNamespace:
    f = lambda *s: np.zeros(s, dtype=np.float64)  # noqa: E731
    i = lambda *s: np.zeros(s, dtype=np.int64)  # noqa: E731
    return SimpleNamespace(
        occ=np.zeros((B, n), np.int8), pref=np.zeros((B, n), np.int8),
        i_drawn=f(B, n), soc=f(B, n), de=f(B, n), cap=f(B, n), rbar=f(B, n), tau=f(B, n), rhat=f(B, n),
        dtrem=i(B, n), b_i=f(B), b_soc=f(B), b_rhat=f(B), step=i(B), day=i(B), episode=i(B),
        env_seed=np.asarray(seeds, dtype=np.uint64).copy(),
        ep_profit=f(B), ep_reward=f(B), ep_missing=f(B), ep_energy=f(B),
        ep_overtime=i(B), ep_declined=i(B), ep_departures=i(B))


def allocate_outs(B: int, n: int, ns: int, obs_len: int) -> SimpleNamespace:
    f = lambda *s: np.zeros(s, dtype=np.float64)  # noqa: E731
    i = lambda *s: np.zeros(s, dtype=np.int64)  # noqa: E731
    return SimpleNamespace(
        obs=f(B, obs_len), reward=f(B), done=np.zeros(B, np.int8), breakdown=f(B, 10), flows=f(B, 5),
        declined=i(B), arrivals_m=i(B), dep_n=i(B), dep_port=i(B, n), dep_missing=f(B, n),
        dep_overtime=i(B, n), dep_early=i(B, n), dep_pref=i(B, n), dep_cap=f(B, n), dep_soc=f(B, n),
        term_overtime=i(B), ep_stats=f(B, 8), i_att=f(B, ns), i_used=f(B, ns), delivered=f(B, n),
        b_delivered=f(B), scratch=f(B, ns))


def _ref_tables(t: StepTables) -> SimpleNamespace:
    """StepTables with the integer dtypes CySimCore's memoryviews expect (_kernel.pyx:85-100)."""
    d = {k: v for k, v in vars(t).items() if not k.startswith("_")}
    for k in ("kind", "order", "node_ptr", "node_leaf", "node_order"):
        d[k] = np.ascontiguousarray(d[k], dtype=np.int64)
    d["weekday"] = np.ascontiguousarray(d["weekday"], dtype=np.int8)
    return SimpleNamespace(**d)


class _OracleCore:
    name = "oracle"

    def __init__(self, t: StepTables, s, o, threads: int):
        self.lib = load_oracle()
        self.tc = t.as_ctypes()
        self.t = t
        self.sc = _State(**{k: getattr(s, k).ctypes.data for k, _ in _State._fields_})
        self.oc = _Outs(**{k: getattr(o, k).ctypes.data for k, _ in _Outs._fields_})
        self.s, self.o, self.threads = s, o, threads

    def reset_env(self, b: int, episode: int) -> None:
        self.lib.vyo_reset_env(C.byref(self.tc), C.byref(self.sc), C.byref(self.oc), b, episode)

    def step_range(self, b0: int, b1: int, a: np.ndarray) -> None:
        self.lib.vyo_step_range(C.byref(self.tc), C.byref(self.sc), C.byref(self.oc), b0, b1, a.ctypes.data)

    def step_all(self, a: np.ndarray) -> None:
        self.lib.vyo_step_parallel(C.byref(self.tc), C.byref(self.sc), C.byref(self.oc), len(a),
                                   a.ctypes.data, self.threads)

    def reset_all(self, first: bool) -> None:
        self.lib.vyo_reset_parallel(C.byref(self.tc), C.byref(self.sc), C.byref(self.oc), len(self.s.step),
                                    int(first), self.threads)

    def step_all_autoreset(self, a: np.ndarray) -> None:
        self.lib.vyo_step_parallel_autoreset(C.byref(self.tc), C.byref(self.sc), C.byref(self.oc), len(a),
                                             a.ctypes.data, self.threads)


class _RefCore:
    """The reference's CySimCore on our arrays; worker threads like engine.py:446-456."""

    name = "ref"

    def __init__(self, t: StepTables, s, o, threads: int):
        self.core = _load_ref().CySimCore(_ref_tables(t), s, o)
        self.threads = threads
        self._pool = None
        if threads > 1:
            from concurrent.futures import ThreadPoolExecutor

            self._pool = ThreadPoolExecutor(threads)

    def reset_env(self, b: int, episode: int) -> None:
        self.core.reset_env(b, episode)

    def step_range(self, b0, b1, a) -> None:
        self.core.step_range(b0, b1, a)

    def step_all(self, a: np.ndarray) -> None:
        B = len(a)
        if self._pool is None:
            self.core.step_range(0, B, a)
            return
        cuts = np.linspace(0, B, self.threads + 1).astype(int)
        futs = [self._pool.submit(self.core.step_range, cuts[w], cuts[w + 1], a)
                for w in range(self.threads) if cuts[w] < cuts[w + 1]]
        for f in futs:
            f.result()


class HostBatch:
    """Reference-semantics batch of envs stepped on the CPU (the checker)."""

    def __init__(self, tables: StepTables, batch_size: int, master_seed: int = 0, env_seeds=None,
                 auto_reset: bool = True, core: str = "oracle", threads: int = 1):
        self.t = tables
        self.batch_size = B = batch_size
        self.auto_reset = auto_reset
        if env_seeds is None:  # split_seed(master, i) for every row, vectorised
            env_seeds = vstream_key(master_seed, np.arange(B, dtype=np.int64))
        self.states = allocate_state(B, tables.n_ports, env_seeds)
        self.outs = allocate_outs(B, tables.n_ports, tables.n_slots, tables.obs_len)
        cls = {"oracle": _OracleCore, "ref": _RefCore}[core]
        self.core = cls(tables, self.states, self.outs, threads)
        self._needs_reset = True

    @property
    def action_size(self) -> int:
        return self.t.n_ports + 1

    def reseed(self, master_seed: int) -> np.ndarray:
        self.states.env_seed[:] = [split_seed(master_seed, i) for i in range(self.batch_size)]
        self._needs_reset = True
        return self.reset()

    def reset(self) -> np.ndarray:
        if hasattr(self.core, "reset_all"):
            self.core.reset_all(self._needs_reset)
        else:
            for b in range(self.batch_size):
                self.core.reset_env(b, 0 if self._needs_reset else int(self.states.episode[b]) + 1)
        self._needs_reset = False
        return self.outs.obs.copy()

    def step(self, actions):
        if self._needs_reset:
            raise EpisodeDone("call reset() before step()")
        a = np.ascontiguousarray(actions, dtype=np.int64)
        if a.shape != (self.batch_size, self.action_size):
            raise ValueError(f"actions shape must be {(self.batch_size, self.action_size)}, got {a.shape}")
        if a.min() < 0 or a.max() > 2 * self.t.k:
            raise ValueError(f"action indices must be in [0, {2 * self.t.k}]")
        if not self.auto_reset and (self.states.step >= self.t.episode_steps).any():
            raise EpisodeDone("an episode is done and auto_reset is off")
        self.core.step_all(a)
        dones = self.outs.done.astype(bool)
        if self.auto_reset:
            for b in np.nonzero(dones)[0]:
                self.core.reset_env(int(b), int(self.states.episode[b]) + 1)
        return self.outs.obs.copy(), self.outs.reward.copy(), dones

    def step_inplace(self, actions: np.ndarray) -> None:
        """step() for large batches: int64 [B, N+1] actions, no validation and no
        copies (outputs stay in self.outs); done rows are reset inside the
        oracle's worker threads (core="oracle" only)."""
        if self.auto_reset:
            self.core.step_all_autoreset(actions)
        else:
            self.core.step_all(actions)


class HostRandomPolicy:
    """RandomPolicy (policies.py:51-73) with the oracle's C draw loop."""

    def __init__(self, seed: int, n_ports: int, k: int, rows, threads: int = 1):
        self.n_slots, self.hi = n_ports + 1, 2 * k + 1
        rows = rows if isinstance(rows, range) else list(rows)
        self.keys = vstream_key(seed, np.asarray(rows, dtype=np.int64), PHASE_POLICY)
        self.threads = threads
        self._out = None

    def actions(self, reuse: bool = False) -> np.ndarray:
        """Next call's actions; reuse=True writes into one persistent buffer."""
        out = self._out if reuse and self._out is not None else np.empty((len(self.keys), self.n_slots), np.int64)
        if reuse:
            self._out = out
        load_oracle().vyo_random_actions_parallel(self.keys.ctypes.data, len(self.keys), self.n_slots, self.hi,
                                                  out.ctypes.data, self.threads)
        return out
