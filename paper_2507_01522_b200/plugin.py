"""The reference-side plugin: a stepping core for voltyard's own ``BatchEnv``.

The reference binds its stepping core through a registry
(``make_core(tables, states, outs, backend)``, backends/__init__.py:43-47);
a core has a ``name`` and two methods, ``reset_env(b, episode)``
(_kernel.pyx:239-261) and ``step_range(b0, b1, actions)`` (_kernel.pyx:275-279),
and works in place on the engine's host arrays (``StateArrays`` /
``StepOutputs``, engine.py:221-336).  ``CudaSimCore`` is that core over the
sm_100a kernels, so the reference's *unmodified* ``BatchEnv`` (validation,
worker split, auto-reset loop, infos) runs on the GPU:

    import voltyard
    from paper_2507_01522_b200 import plugin
    plugin.register(voltyard)            # adds backend "cuda"
    env = voltyard.BatchEnv(cfg, station, ds, batch_size=B, backend="cuda")

Batching.  The engine calls ``reset_env`` once per env, in index order
(``reset``: every row; auto-reset: the rows the step finished).  The core
queues those calls and resets the queued rows in ONE masked launch
(``vy_reset_episodes``) as soon as the sweep is complete — at the last of the
rows the previous step finished, at row B-1 of a full sweep, or at the next
``step_range`` — so the engine's ``outs.obs.copy()`` right after its loop
already reads the reset observations.  ``step_range`` calls from the engine's
worker threads (``workers > 1``, engine.py:446-456) are gathered until they
cover [0, B) and then stepped as one launch; results do not depend on the
worker count (the reference's own contract, tests/test_engine.py:78-86).

Mirroring (``mirror=``, or the VOLTYARD_CUDA_MIRROR environment variable):

* ``"full"`` (default, the exact drop-in): the host arrays stay the source of
  truth, exactly as with CySimCore.  Each launch uploads the host state
  (in the reference layout; cap / rbar / tau map onto the car-profile table,
  unseen cars are registered like the reference tests' ``inject_car``), runs
  the generic float64 kernel with the info block, and writes back every state
  slot and every output the reference kernel writes (departure records only
  for the first ``dep_n`` entries, ``ep_stats`` only for finished rows —
  what the reference leaves untouched stays untouched).
* ``"outputs"``: the device state is the source of truth.  Only what
  ``BatchEnv.step(collect_infos=False)`` reads comes back — obs, reward, done,
  ``term_overtime``, finished rows' ``ep_stats`` and the ``step`` / ``day`` /
  ``episode`` counters; host writes to other state slots are not seen.  This
  is the throughput mode of the reference API (``throughput_probe`` runs with
  infos off, engine.py:541-545).
"""

from __future__ import annotations

import os
import threading

import numpy as np
import torch

from . import _native as nat
from .batch import BatchEnv
from .streams import PHASE_ARRIVALS, vstream_key
from .tables import StepTables, build_tables_from_kernel_tables

BACKEND_CUDA = "cuda"
_STATE_F64 = ("i_drawn", "soc", "de")
_ENV_F64 = ("b_i", "b_soc", "ep_profit", "ep_reward", "ep_missing", "ep_energy")
_ENV_I32 = ("ep_overtime", "ep_declined", "ep_departures")
_INFO_ALWAYS = ("breakdown", "flows", "declined", "arrivals_m", "dep_n", "i_att", "i_used", "delivered",
                "b_delivered")
_DEP = ("dep_port", "dep_missing", "dep_overtime", "dep_early", "dep_pref", "dep_cap", "dep_soc")


class CudaSimCore:
    """core protocol of backends/_kernel.pyx:119-279 over the CUDA kernels."""

    name = BACKEND_CUDA

    def __init__(self, tables, states, outs, mirror: str | None = None, device=None):
        mirror = (mirror or os.environ.get("VOLTYARD_CUDA_MIRROR", "full")).lower()
        if mirror not in ("full", "outputs"):
            raise ValueError(f"mirror must be 'full' or 'outputs', got {mirror!r}")
        self.mirror = mirror
        t = tables if isinstance(tables, StepTables) else build_tables_from_kernel_tables(tables)
        self.t, self.s, self.o = t, states, outs
        self.B = B = len(states.step)
        self.env = BatchEnv(None, None, None, batch_size=B, env_seeds=np.asarray(states.env_seed, np.uint64),
                            auto_reset=False, obs_dtype=torch.float64, device=device, tables=t)
        self.env.outs.ensure_info()
        self.env._bind()
        self.dev = self.env.device
        self._kind = np.asarray(t.kind, dtype=np.int64)
        self._pids: dict = {}
        self._pending = np.full(B, -1, dtype=np.int64)  # queued reset_env episode per row (-1: none)
        self._expect: np.ndarray | None = None  # rows the last step finished (the engine resets them next)
        self._cover = np.zeros(B, dtype=bool)
        self._stage = np.zeros((B, t.n_ports + 1), dtype=np.int64)
        self._lock = threading.Lock()
        self._synced = False  # "outputs" mode: device state initialised from the host arrays

    # -- reference layout <-> device layout ----------------------------------------

    def _profile_id(self, cap: float, rbar: float, tau: float, kind: int) -> int:
        key = (cap, rbar, tau, kind)
        pid = self._pids.get(key)
        if pid is None:
            t = self.t
            for c in range(t.n_cat):  # a catalogue car (_kernel.pyx:497-502)
                r = t.cat_rdc[c] if kind == 1 else t.cat_rac[c]
                if t.cat_cap[c] == cap and t.cat_tau[c] == tau and r == rbar:
                    pid = c
                    break
            if pid is None:  # a car placed by hand (tests/helpers.py:163-189)
                pid = int(self.env._lib.vy_add_profile(self.env._h, float(cap), float(rbar), float(rbar), float(tau)))
                if pid < 0:
                    raise ValueError(self.env._lib.vy_last_error().decode())
            self._pids[key] = pid
        return pid

    def _dev(self, a: np.ndarray, dtype=None) -> torch.Tensor:
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.to(self.dev, dtype=dtype) if dtype is not None else t.to(self.dev)

    def _upload_state(self) -> None:
        """Host StateArrays (engine.py:221-279) -> device SoA (vy_state)."""
        s, d, B = self.s, self.env.states, self.B
        occ = s.occ.astype(bool)
        prof = np.zeros(occ.shape, dtype=np.int64)
        if occ.any():
            keys = np.stack([s.cap[occ], s.rbar[occ], s.tau[occ], np.broadcast_to(self._kind, occ.shape)[occ]], 1)
            uniq, inv = np.unique(keys, axis=0, return_inverse=True)
            ids = np.array([self._profile_id(float(u[0]), float(u[1]), float(u[2]), int(u[3])) for u in uniq])
            prof[occ] = ids[inv.reshape(-1)]
        meta = (occ.astype(np.int64) | ((s.pref.astype(np.int64) & 1) << 1) | (prof << 2)).astype(np.uint8)
        for name, src in (("port_i", s.i_drawn), ("port_soc", s.soc), ("port_de", s.de)):
            getattr(d, name)[:, :B].copy_(self._dev(src).T)
        d.port_dtrem[:, :B].copy_(self._dev(s.dtrem, torch.int16).T)
        d.port_meta[:, :B].copy_(self._dev(meta).T)
        for name in ("step", "day", "episode"):
            getattr(d, name)[:B].copy_(self._dev(getattr(s, name), torch.int32))
        seeds = np.ascontiguousarray(s.env_seed, dtype=np.uint64)
        d.env_seed[:B].copy_(self._dev(seeds.view(np.int64)))
        # arrival-stream prefix of the current episode: stream_key(seed, episode, 1) (_kernel.pyx:461)
        akey = vstream_key(seeds, np.asarray(s.episode, dtype=np.int64), PHASE_ARRIVALS)
        d.akey[:B].copy_(self._dev(akey.view(np.int64)))
        for name in _ENV_F64:
            getattr(d, name)[:B].copy_(self._dev(getattr(s, name)))
        for name in _ENV_I32:
            getattr(d, name)[:B].copy_(self._dev(getattr(s, name), torch.int32))

    def _download_state(self) -> None:
        st = self.env.reference_state()
        for k, v in st.items():
            if k != "env_seed":
                getattr(self.s, k)[...] = v

    def _download_counters(self) -> None:
        d, s, B = self.env.states, self.s, self.B
        for name in ("step", "day", "episode"):
            getattr(s, name)[...] = getattr(d, name)[:B].cpu().numpy()

    def _sync_in(self, seeds: bool = False) -> None:
        if self.mirror == "full" or not self._synced:
            self._upload_state()
            self._synced = True
        elif seeds:  # reseed() rewrites the host seeds before its reset sweep (engine.py:407-412)
            s = np.ascontiguousarray(self.s.env_seed, dtype=np.uint64)
            self.env.states.env_seed[: self.B].copy_(self._dev(s.view(np.int64)))

    # -- core protocol ----------------------------------------------------------------

    def reset_env(self, b: int, episode: int) -> None:
        """_kernel.pyx:239-261, queued; see the module docstring for when it runs."""
        b = int(b)
        if not 0 <= b < self.B:
            raise IndexError(f"env index {b} out of range")
        with self._lock:
            self._pending[b] = int(episode)
            if self._expect is not None:
                self._expect[b] = False
                if not self._expect.any():
                    self._flush_resets()
            elif b == self.B - 1:
                self._flush_resets()

    def step_range(self, b0: int, b1: int, actions) -> None:
        """_kernel.pyx:275-279; slices are gathered until they cover [0, B)."""
        b0, b1 = int(b0), int(b1)
        if not 0 <= b0 <= b1 <= self.B:
            raise IndexError("step range out of bounds")
        if b0 == b1:
            return
        a = np.asarray(actions)
        with self._lock:
            if b0 == 0 and b1 == self.B and not self._cover.any():
                self._step_all(np.ascontiguousarray(a, dtype=np.int64))
                return
            self._stage[b0:b1] = a[b0:b1]
            self._cover[b0:b1] = True
            if self._cover.all():
                self._cover[:] = False
                self._step_all(self._stage)

    # -- launches ----------------------------------------------------------------------

    def _flush_resets(self) -> None:
        rows = self._pending >= 0
        self._expect = None
        if not rows.any():
            return
        env, o = self.env, self.o
        self._sync_in(seeds=True)
        mask = self._dev(rows.astype(np.uint8))
        eps = self._dev(np.where(rows, self._pending, 0), torch.int32)
        flags = nat.F_OUT_F64
        nat.check(env._lib.vy_reset_episodes(env._h, mask.data_ptr(), eps.data_ptr(), flags, env._stream),
                  "vy_reset_episodes")
        o.obs[rows] = env.outs.obs[torch.from_numpy(rows).to(self.dev)].cpu().numpy()
        if self.mirror == "full":
            self._download_state()
        else:
            self._download_counters()
        self._pending[:] = -1

    def _step_all(self, a: np.ndarray) -> None:
        if (self._pending >= 0).any():
            self._flush_resets()
        env, o, B = self.env, self.o, self.B
        self._sync_in()
        act = self._dev(a)
        full = self.mirror == "full"
        flags = nat.F_OUT_F64 | (nat.F_INFOS if full else 0)
        nat.check(env._lib.vy_step(env._h, act.data_ptr(), nat.VY_ACT_I64, a.shape[1], 1, flags, None, env._stream),
                  "vy_step")
        word = np.zeros(1, dtype=np.uint32)
        nat.check(env._lib.vy_poll_error(env._h, 1, env._stream, word.ctypes.data_as(nat.C.POINTER(nat.C.c_uint32))),
                  "vy_poll_error")
        if word[0] & 1:
            raise ValueError(f"action indices must be in [0, {2 * self.t.k}]")
        out = env.outs
        o.obs[...] = out.obs.cpu().numpy()
        o.reward[...] = out.reward.cpu().numpy()
        done = out.done.cpu().numpy().astype(np.int8)
        o.done[...] = done
        fin = done.astype(bool)
        # terminal overtime of finished rows, 0 for the others (_kernel.pyx:553-570)
        o.term_overtime[...] = np.where(fin, out.term_overtime[:B].cpu().numpy(), 0)
        if fin.any():  # the reference writes ep_stats at the episode end only (_kernel.pyx:556-568)
            o.ep_stats[fin] = out.ep_stats[:, :B].cpu().numpy().T[fin]
        if full:
            info = {k: v[..., :B].cpu().numpy() for k, v in out.info.items()}
            for k in _INFO_ALWAYS:
                v = info[k]
                getattr(o, k)[...] = v.T if v.ndim == 2 else v
            # departure records: only the first dep_n entries are written (_kernel.pyx:426-458)
            keep = np.arange(self.t.n_ports)[None, :] < info["dep_n"][:, None]
            for k in _DEP:
                dst = getattr(o, k)
                dst[keep] = info[k].T[keep]
            self._download_state()
        else:
            self._download_counters()
        self._expect = fin.copy() if fin.any() else None

    def close(self) -> None:
        self.env.close()


def make_core(tables, states, outs, backend: str | None = None, **kw):
    """The registry entry point (backends/__init__.py:43-47) for backend "cuda"."""
    return CudaSimCore(tables, states, outs, **kw)


def register(voltyard) -> None:
    """Make ``backend="cuda"`` selectable in an installed reference package
    without editing it: wraps ``resolve_backend`` / ``make_core`` of
    ``voltyard.backends`` and the names ``voltyard.engine`` imported from it
    (engine.py:22).  Other backend names reach the original functions."""
    import importlib

    backends = importlib.import_module(voltyard.__name__ + ".backends")
    engine = importlib.import_module(voltyard.__name__ + ".engine")
    if getattr(backends, "_cuda_registered", False):
        return
    orig_resolve, orig_make, orig_avail = backends.resolve_backend, backends.make_core, backends.available_backends

    def resolve_backend(name=None):
        if name is None:
            name = os.environ.get("VOLTYARD_BACKEND")
        if name is not None and name.lower() == BACKEND_CUDA:
            return BACKEND_CUDA
        return orig_resolve(name)

    def make_core_any(tables, states, outs, backend=None):
        if resolve_backend(backend) == BACKEND_CUDA:
            return CudaSimCore(tables, states, outs)
        return orig_make(tables, states, outs, backend)

    def available_backends():
        return tuple(orig_avail()) + (BACKEND_CUDA,)

    for mod in (backends, engine):
        if hasattr(mod, "resolve_backend"):
            mod.resolve_backend = resolve_backend
        if hasattr(mod, "make_core"):
            mod.make_core = make_core_any
    backends.available_backends = available_backends
    backends._cuda_registered = True


__all__ = ["CudaSimCore", "make_core", "register", "BACKEND_CUDA"]
