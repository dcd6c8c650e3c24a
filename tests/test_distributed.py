"""Multi-process sharding on CPU (gloo, world_size 2).

Each rank steps its shard of the global batch with the CPU oracle (the GPU is
not available here; the sharding plan, global seeding and the statistics
collective are what is under test) and the union must equal the unsharded
run bit for bit; the all_reduced statistics must equal the single-process sums.
"""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_01522_b200 import EnvConfig, default_setup
from paper_2507_01522_b200.sharding import plan, reduce_rollout_stats
from paper_2507_01522_b200.streams import split_seed
from paper_2507_01522_b200.tables import build_tables

GLOBAL, STEPS, MASTER, PSEED = 24, 40, 13, 3


def _run_rows(rows):
    from oracle.harness import HostBatch, HostRandomPolicy

    rc = default_setup(EnvConfig(episode_steps=16), days=20)
    t = build_tables(rc.env, rc.station, rc.dataset)
    hb = HostBatch(t, len(rows), env_seeds=[split_seed(MASTER, i) for i in rows])
    pol = HostRandomPolicy(PSEED, t.n_ports, t.k, rows)
    hb.reset()
    rew, eps = [], []
    for _ in range(STEPS):
        o, r, d = hb.step(pol.actions())
        rew.append(r)
        eps.append(np.where(d, hb.outs.ep_stats[:, 1], 0.0))
    return o, np.array(rew), np.array(eps)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = plan(GLOBAL, world)[rank]
    obs, rew, eps = _run_rows(range(sh.offset, sh.offset + sh.count))
    stats = torch.tensor([rew.sum(), eps.sum(), float(sh.count)], dtype=torch.float64)
    reduce_rollout_stats(stats)
    out[rank] = (sh.offset, obs, rew, stats.numpy())
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_covers_range():
    for world in (1, 2, 3, 8):
        sh = plan(1000, world)
        assert sh[0].offset == 0 and sum(s.count for s in sh) == 1000
        assert all(a.offset + a.count == b.offset for a, b in zip(sh, sh[1:]))


def test_two_rank_shards_equal_single_batch():
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    obs_full, rew_full, eps_full = _run_rows(range(GLOBAL))
    for rank in range(world):
        off, obs, rew, stats = res[rank]
        np.testing.assert_array_equal(obs, obs_full[off:off + len(obs)])
        np.testing.assert_array_equal(rew, rew_full[:, off:off + rew.shape[1]])
        np.testing.assert_allclose(stats, [rew_full.sum(), eps_full.sum(), GLOBAL], rtol=1e-12)


def test_sweep_groups_cover_c5_grid():
    from paper_2507_01522_b200.hetero import sweep_groups

    gs = sweep_groups(total_envs=1 << 16, days=3)
    assert len(gs) == 36 and sum(g.batch_size for g in gs) == 1 << 16
    assert len({g.name.split("/")[0] for g in gs}) == 3 and len({g.name.split("/")[1] for g in gs}) == 4
    assert {g.station.n_ports for g in gs} == {8, 16}


def _grad_worker(rank, world, port, out):
    """PPO's gradient all-reduce (ppo.allreduce_mean_) on gloo: different
    per-rank gradients become their mean on every rank, and the Adam step that
    follows leaves identical weights everywhere."""
    from paper_2507_01522_b200.ppo import ActorCritic, allreduce_mean_

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(rank)  # different initial weights: the broadcast must fix them
    net = ActorCritic(105, 17, 21, 64)
    for p in net.parameters():
        dist.broadcast(p.data, 0)
    opt = torch.optim.Adam(net.parameters(), lr=1e-3)
    g = torch.Generator().manual_seed(100 + rank)  # rank-specific data
    x = torch.randn(64, 105, generator=g)
    logits, v = net(x)
    (logits.square().mean() + v.square().mean()).backward()
    local = [p.grad.clone() for p in net.parameters()]
    allreduce_mean_([p.grad for p in net.parameters()], world)
    opt.step()
    out[rank] = ([t.numpy() for t in local], [p.grad.numpy().copy() for p in net.parameters()],
                 [p.data.numpy().copy() for p in net.parameters()])
    dist.destroy_process_group()


def test_two_rank_ppo_gradient_mean_and_identical_weights():
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_grad_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    local0, mean0, w0 = res[0]
    local1, mean1, w1 = res[1]
    for a, b, m0, m1 in zip(local0, local1, mean0, mean1):
        assert not np.array_equal(a, b)
        np.testing.assert_allclose(m0, (a + b) / 2, rtol=1e-6, atol=1e-7)
        np.testing.assert_array_equal(m0, m1)
    for a, b in zip(w0, w1):
        np.testing.assert_array_equal(a, b)
