"""Heterogeneous station configurations on one GPU (BASELINE config C5).

The reference requires one (config, station, dataset) per batch
(engine.py:370).  ``HeteroBatch`` batches many: each group is a
regular BatchEnv (own tables, own handle; the lean step kernel when the
group's config allows it — group sizes are whole 32-env tiles for that),
groups are launched costliest first (largest tree, then most ports),
round-robin over CUDA streams, so the per-group grids run concurrently, fill
the GPU and the slowest groups do not form the step's tail (each group's launches stay ordered on its
stream; a step joins all streams back into the caller's), and each group's
persistent grid is shaped for sharing (``tiles_per_warp``).  Env seeds and
RandomPolicy rows use one global index space across groups (group g's envs
are global indices offset_g .. offset_g + B_g - 1), so a group's trajectory is
bit-identical to a standalone BatchEnv with that global_offset — which is
what the tests check.

``MultiStep`` (``HeteroBatch.multi_random_step``) is the one-launch form: a
multi handle (vy_multi_create) stacks the groups' Params in device memory and
one persistent kernel (k_step_multi) steps every group, global tile t mapped
to its group by the per-tile config index and each
distinct table set staged once per CTA; the outputs equal the per-group
launches bit for bit.

``sweep_groups`` builds the C5 sweep: regions {eu, us, world} x scenarios
{highway, residential, work, shopping} x traffic {low, medium, high}, station
presets rotating over single / multi / nested layouts.
"""

from __future__ import annotations

import ctypes as C
import itertools
from dataclasses import dataclass

import torch

from . import _native as nat
from .batch import BatchEnv, DeviceRandomPolicy
from .envconfig import EnvConfig
from .exogenous import REGIONS, SCENARIOS, TRAFFIC_FACTORS, Dataset, generate_synthetic_defaults
from .station import StationTree, preset_station


@dataclass
class Group:
    name: str
    config: EnvConfig
    station: StationTree
    dataset: Dataset
    batch_size: int


_LAYOUTS = (("single_type", 0, 8), ("multi_type", 6, 10), ("nested_splitters", 4, 12))


def sweep_groups(total_envs: int, days: int = 365, seed: int = 0) -> list[Group]:
    """36 (region, scenario, traffic) combinations splitting ``total_envs``."""
    combos = list(itertools.product(REGIONS, SCENARIOS, TRAFFIC_FACTORS))
    # whole 32-env warp tiles per group (when the total allows): the lean step
    # kernel stages each tile's uint8 action rows, which needs B % 32 == 0
    per = total_envs // len(combos)
    if per >= 32:
        per -= per % 32
    groups = []
    for gi, (region, scen, traffic) in enumerate(combos):
        layout, ac, dc = _LAYOUTS[gi % len(_LAYOUTS)]
        ds = generate_synthetic_defaults(scen, traffic, region, seed=seed, days=days)
        groups.append(Group(f"{region}/{scen}/{traffic}/{layout}", EnvConfig(), preset_station(layout, ac, dc), ds,
                            per if gi < len(combos) - 1 else total_envs - per * (len(combos) - 1)))
    return groups


class HeteroBatch:
    def __init__(self, groups: list[Group], master_seed: int = 0, global_offset: int = 0, device=None,
                 policy_seed: int | None = None, n_streams: int = 12, tiles_per_warp: int = 3,
                 longest_first: bool = True):
        self.groups = groups
        self.streams = [torch.cuda.Stream(device=device) for _ in range(max(1, n_streams))]
        self.envs: list[BatchEnv] = []
        self.policies: list[DeviceRandomPolicy] = []
        off = global_offset
        for g in groups:
            env = BatchEnv(g.config, g.station, g.dataset, batch_size=g.batch_size, master_seed=master_seed,
                           global_offset=off, device=device)
            env.set_tiles_per_warp(tiles_per_warp)  # groups overlap on streams: fewer, longer-lived warps each
            self.envs.append(env)
            if policy_seed is not None:
                pol = DeviceRandomPolicy(policy_seed, env.n_ports, g.config.discretization_k)
                pol.bind(range(off, off + g.batch_size))
                self.policies.append(pol)
            off += g.batch_size
        self.total = off - global_offset
        # launch order: the costliest groups first (bigger trees, then more
        # ports, then more envs) so they do not form the step's tail
        cost = [(e.tables.n_nodes, e.n_ports, g.batch_size) for e, g in zip(self.envs, groups)]
        self._order = sorted(range(len(groups)), key=lambda i: cost[i], reverse=True) if longest_first \
            else list(range(len(groups)))

    def reset(self) -> list[torch.Tensor]:
        return [e.reset(as_numpy=False) for e in self.envs]

    def _fan_out(self, fn):
        """Run fn(i) for every group on its stream; join into the current stream."""
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        out = [None] * len(self.envs)
        for p, i in enumerate(self._order):
            with torch.cuda.stream(self.streams[p % len(self.streams)]):
                out[i] = fn(i)
        for s in self.streams:
            cur.wait_stream(s)
        return out

    def step(self, actions: list[torch.Tensor]):
        """One step of every group; returns per-group (obs, reward, done)."""
        def one(i):
            o, r, d, _ = self.envs[i].step(actions[i], collect_infos=False)
            return o, r, d

        return self._fan_out(one)

    def random_step(self):
        """One step of every group with its device RandomPolicy actions (drawn
        inside each group's step kernel, vy_step_random)."""
        def one(i):
            o, r, d, _ = self.envs[i].step_random(self.policies[i])
            return o, r, d

        return self._fan_out(one)

    def graph_random_step(self) -> None:
        """random_step replayed from a captured CUDA graph: the group launches
        and their stream fork/join cost one graph launch.  Actions come from the
        device-counter RandomPolicy (vy_random_actions_dev), so every replay
        draws the next call; the host-side lockstep clocks and call counters are
        advanced here because a replay runs no host code.  One fused
        policy+step kernel per group."""
        if getattr(self, "_graph", None) is None:
            def one(i):
                o, r, d, _ = self.envs[i].step_random(self.policies[i], device_counter=True)
                return o, r, d

            clocks = [e._t for e in self.envs]
            # warm-up (creates the device counters) then capture
            self._fan_out(one)
            for p in self.policies:
                p.calls += 1
            clocks = [e._t for e in self.envs]
            self._graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self._graph):
                self._fan_out(one)
            for e, c in zip(self.envs, clocks):
                e._t = c  # capture did not execute
            return  # the warm-up was this call's step
        self._graph.replay()
        for p in self.policies:
            p.calls += 1
        for e in self.envs:
            if e._t is not None:
                e._t = (e._t + 1) % e.tables.episode_steps

    # ---- one launch per step over all groups (k_step_multi) -------------
    def _multi_handle(self):
        if getattr(self, "_multi", None) is None:
            if len(self.policies) != len(self.envs):
                raise ValueError("multi_random_step needs a policy_seed (device RandomPolicy per group)")
            n = len(self.envs)
            hs = (C.c_void_p * n)(*[e._h for e in self.envs])
            seeds = (C.c_uint64 * n)(*[p.seed & ((1 << 64) - 1) for p in self.policies])
            idx = (C.c_int64 * n)(*[p.index0 for p in self.policies])
            out = C.c_void_p()
            lib = self.envs[0]._lib
            nat.check(lib.vy_multi_create(hs, n, seeds, idx, C.byref(out)), "vy_multi_create")
            self._multi = out
        return self._multi

    def multi_info(self) -> dict:
        """Spec mode, distinct table sets, warps per CTA and grid of the one-launch step."""
        v = (C.c_int32 * 4)()
        nat.check(self.envs[0]._lib.vy_multi_info(self._multi_handle(), v), "vy_multi_info")
        return {"mode": v[0], "profile_sets": v[1] // 16, "station_sets": v[1] % 16, "warps_per_cta": v[2],
                "grid": v[3]}

    def multi_random_step(self, device_counter: torch.Tensor | None = None) -> None:
        """One step of every group with its device RandomPolicy rows as ONE
        kernel launch (k_step_multi); outputs land in each group's buffers
        (``self.envs[g].outs``), bit-identical to ``random_step``.  With
        ``device_counter`` (int64 [2] on the device, zeroed) the policy call
        index is read from device memory and advanced by the kernel (CUDA
        graph replay); the host clocks and call counters advance here."""
        for e in self.envs:
            if e._needs_reset:
                raise nat.EpisodeDone("call reset() before step()")
        m = self._multi_handle()
        lib = self.envs[0]._lib
        call = 0 if device_counter is not None else self.policies[0].calls
        if device_counter is None and any(p.calls != call for p in self.policies):
            raise ValueError("group policies are at different call indices")
        ptr = device_counter.data_ptr() if device_counter is not None else None
        nat.check(lib.vy_multi_step_random(m, call, ptr, torch.cuda.current_stream().cuda_stream), "vy_multi_step")
        for p in self.policies:
            p.calls += 1
        for e in self.envs:
            e._advance_clock()

    def graph_multi_step(self) -> None:
        """multi_random_step replayed from a captured CUDA graph (one kernel
        node); the device counter carries the RandomPolicy call index."""
        if getattr(self, "_mgraph", None) is None:
            self._mcounter = torch.zeros(2, dtype=torch.int64, device=self.envs[0].outs.obs.device)
            self._mcounter[0] = self.policies[0].calls
            self.multi_random_step(self._mcounter)  # warm-up: this call's step
            clocks = [e._t for e in self.envs]
            calls = [p.calls for p in self.policies]
            self._mgraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self._mgraph):
                self.multi_random_step(self._mcounter)
            for e, c in zip(self.envs, clocks):
                e._t = c  # capture did not execute
            for p, c in zip(self.policies, calls):
                p.calls = c
            return
        self._mgraph.replay()
        for p in self.policies:
            p.calls += 1
        for e in self.envs:
            e._advance_clock()

    def kernels_per_step(self) -> int:
        return len(self.envs)

    def launch_count(self) -> int:
        return sum(e.launch_count() for e in self.envs)

    def close(self) -> None:
        if getattr(self, "_multi", None) is not None:
            self.envs[0]._lib.vy_multi_destroy(self._multi)
            self._multi = None
        for e in self.envs:
            e.close()
